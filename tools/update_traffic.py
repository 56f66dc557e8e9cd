"""Write the cfg3 / cfg5q6 entries of profiles/traffic.json from one round-profile tag
(tools/round_profiles_r02.sh TAG): DRAM bytes per launch of the timed kernel, predicated-on
FP64 thread instructions and DMMA instructions per DoF, the profile files and the build hash.
python tools/update_traffic.py TAG   (reads profiles/TAG_*_metrics.csv, profiles/TAG_build.txt)"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
P = os.path.join(ROOT, "profiles")


def metrics(path):
    out, h = {}, None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            out["kernel"] = d["Kernel Name"]
            out[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


build = open(os.path.join(P, f"{tag}_build.txt")).read().strip()
tj = os.path.join(P, "traffic.json")
t = json.load(open(tj))
fp64_keys = ["sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
             "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]

m = metrics(os.path.join(P, f"{tag}_halo_cfg3_metrics.csv"))
n3 = 16974593
b3 = int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
prev = t.get("cfg3", {})
t["cfg3"] = {
    "bytes_per_launch": b3,
    "kernels": {"k_apply_halo<true>": b3},
    "source": [f"profiles/{tag}_halo_cfg3_metrics.csv", f"profiles/{tag}_halo_cfg3_ncu.txt"],
    "build": build,
    "fp64_instr_per_dof": round(sum(m[k] for k in fp64_keys) / n3, 2),
    "fp64_instr_note": "predicated-on DFMA + DADD + DMUL thread instructions of one k_apply_halo<true> launch "
                       "(the kernel the bench times; no init kernel) / 16,974,593 DoFs",
    "previous": prev.get("previous", ""),
}

m = metrics(os.path.join(P, f"{tag}_tc_cfg5q6_metrics.csv"))
n6 = 3630961153
b6 = int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
t["cfg5q6"] = {
    "bytes_per_launch": b6,
    "kernels": {"k_apply_tc<6>": b6},
    "source": [f"profiles/{tag}_tc_cfg5q6_metrics.csv", f"profiles/{tag}_tc_q6_64_ncu.txt"],
    "build": build,
    "fp64_instr_per_dof": round(sum(m[k] for k in fp64_keys) / n6, 2),
    # sm__ops_path_tensor_src_fp64 counts 2 per FMA; one m8n8k4 f64 DMMA = 256 FMA
    "dmma_per_dof": round(m["sm__ops_path_tensor_src_fp64.sum"] / 512 / n6, 4),
    "fp64_instr_note": "predicated-on DFMA + DADD + DMUL thread instructions and DMMA instructions "
                       "(sm__ops_path_tensor_src_fp64 / 512) of one k_apply_tc<6> launch / 3,630,961,153 DoFs; "
                       "the timed region also holds the dst zeroing kernel (~4.5 ms, 29 GB written)",
}
json.dump(t, open(tj, "w"), indent=1)
print(json.dumps({k: t[k] for k in ("cfg3", "cfg5q6")}, indent=1))
