for L in HALO_NOLOAD HALO_ONLY_CONS; do
  echo $L; MF_LIB_PATH=$PWD/paper_1910_13247_b200/lib_$L.so timeout 60 python tools/time_apply.py --shape 32,32,256 --degree 4 --variant halo --reps 30 2>&1 | tail -1
done
