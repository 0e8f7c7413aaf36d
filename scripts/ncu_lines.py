"""Per-CUDA-source-line instruction and stall-sample shares from an ncu report.

    python scripts/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s, i_i = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if r and r[0] and r[0].isdigit() and len(r) > i_i:
        try:
            lines.append((int(r[0]), r[1].strip()[:70], float(r[i_s] or 0), float(r[i_i] or 0)))
        except ValueError:
            pass
S = sum(x[2] for x in lines) or 1
I = sum(x[3] for x in lines) or 1
print(f"total warp-instr {I:.0f}  samples {S:.0f}")
for ln, src, s, i in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{ln:5d} instr {100 * i / I:5.1f}% stall {100 * s / S:5.1f}%  {src}")
