"""Summarise an ncu report: key throughput / pipe / stall metrics (run here, no GPU)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[head.index("Kernel Name")] if "Kernel Name" in head else "?"
        print("kernel:", name[:80])
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        stalls = [(k, float(v)) for k, v in d.items()
                  if k.startswith("smsp__average_warp_latency_issue_stalled") or
                  (k.startswith("smsp__warp_issue_stalled_") and k.endswith("_per_warp_active.pct"))]
        stalls = sorted([s for s in stalls if s[1] > 0], key=lambda s: -s[1])[:10]
        for k, v in stalls:
            print(f"  stall {k.replace('smsp__warp_issue_stalled_', '')} = {v:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
