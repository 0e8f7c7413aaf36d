"""One-file text summary of an ncu --set full report (key metrics + per-line table).

    python scripts/ncu_summary.py report.ncu-rep "header" > profiles/rNN_ncu_X.txt
"""
import csv
import io
import subprocess
import sys

rep, head = sys.argv[1], sys.argv[2]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
print("# " + head)
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
print("# kernel: " + rows[1][h.index("Kernel Name")][:160])
want = ["Memory Throughput", "DRAM Throughput", "Duration", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Mem Busy", "Max Bandwidth", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy"]
seen = set()
for r in rows[1:]:
    n = r[h.index("Metric Name")]
    if n in want and n not in seen:
        seen.add(n)
        print(f"{n:<45} {r[h.index('Metric Value')]:>14} {r[h.index('Metric Unit')]}")
rr = list(csv.reader(io.StringIO(raw)))
H, U, V = rr[0], rr[1], rr[2]
for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]:
    if key in H:
        i = H.index(key)
        print(f"{key:<45} {V[i]:>14} {U[i]}")
for i, n in enumerate(H):
    if "warps_issue_stalled" in n and "per_issue_active" in n:
        try:
            if float(V[i]) > 0.2:
                print(f"{n:<75} {V[i]}")
        except ValueError:
            pass
print("# per source line (share of executed warp-instructions / of stall samples)")
sys.stdout.flush()
subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"), rep, "20"])
