"""Selected raw metrics of ncu --set full reports -> JSON (profiles/rNN_ncu_full.json).
usage: python tools/ncu_summary.py out.json name=report.ncu-rep [name=report.ncu-rep ...]"""
import csv, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "launch__shared_mem_per_block_static", "launch__occupancy_limit_registers",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__cluster_dim_x"]
out = {}
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                          text=True).stdout.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out[name] = {k: [vals[hdr.index(k)], units[hdr.index(k)]] for k in KEYS if k in hdr}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps({k: v.get("gpu__time_duration.sum") for k, v in out.items()}))
