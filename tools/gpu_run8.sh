for L in HALO_NB2_HALO_NS4 HALO_PF2 HALO_PF4 HALO_NB2_HALO_NS4_HALO_PF2; do
  echo $L; for sh in 64,64,64 32,32,256; do MF_LIB_PATH=$PWD/paper_1910_13247_b200/lib_$L.so timeout 60 python tools/time_apply.py --shape $sh --degree 4 --variant halo --reps 30 2>&1 | tail -1; done
done
