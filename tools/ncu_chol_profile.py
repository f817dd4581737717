"""Summarise one `ncu --set full` capture of k_chol_tiles into profiles/.

usage: python tools/ncu_chol_profile.py <report.ncu-rep> <config> <systems_per_launch> <capture note>
writes profiles/ncu_chol_cfg<config>.json (read by bench.py for roofline.traffic)
and prints a text summary (metrics + stall reasons by source line).
"""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.sum",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "launch__grid_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h, units, v = rows[0], rows[1], rows[2]
    return {n: (v[i], units[i]) for i, n in enumerate(h)}


def main():
    rep, cfg, spl, note = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    m = raw(rep)
    res = {}
    for k in METRICS:
        if k in m:
            res[k] = f"{m[k][0]} {m[k][1]}".strip()
    def to_bytes(k):
        val, unit = m[k]
        return float(val.replace(",", "")) * UNITS.get(unit, 1)
    traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    res["systems_per_launch"] = spl
    res["dram_bytes_per_launch"] = int(traffic)
    res["capture"] = note
    path = os.path.join(ROOT, "profiles", f"ncu_chol_cfg{cfg}.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    for k, v in res.items():
        print(f"{k}: {v}")
    objs = sorted(glob.glob(os.path.join(ROOT, "build", "obj", "chol.cu.*.o")), key=os.path.getmtime)
    if objs:
        print("stall samples by source line (tools/ncu_lines.py):")
        sys.stdout.flush()
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, objs[-1],
                        os.environ.get("KERNEL_SYM", "_ZN4slim9k_chol_i8ENS_10CholParamsE")],
                       env=dict(os.environ, TOP="15"))


main()
