"""Key counters and stall reasons of the kernels in an ncu report.

usage: python tools/ncu_keys.py <report.ncu-rep>
"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sectors.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "smsp__warps_active.avg.per_cycle_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__issue_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "smsp__inst_executed_op_shared_atom_dot_cas.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for d in rows[2:]:
        print("==", d[h.index("Kernel Name")][:60])
        for w in WANT:
            if w in h:
                print(f"  {w:62s} {d[h.index(w)]}")
        st = []
        for i, n in enumerate(h):
            if "issue_stalled" in n and n.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(d[i].replace(",", "")), n))
                except ValueError:
                    pass
        for v, n in sorted(st, reverse=True)[:8]:
            print(f"  stall {v:6.2f} "
                  f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")


main()
