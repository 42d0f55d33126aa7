"""Top source lines by warp-stall samples from an ncu report (--import-source).
python tools/ncu_lines.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
src = [r for r in rows if len(r) > 7 and r[0].isdigit()]
tot = sum(int(r[4]) for r in src if r[4].isdigit()) or 1
print("total samples", tot)
for r in sorted(src, key=lambda r: -int(r[4]) if r[4].isdigit() else 0)[:n]:
    print(f"{r[0]:>5} {int(r[4]) * 100 / tot:5.1f}% not-issued={r[5]:>8} inst={r[7]:>12}  {r[1].strip()[:100]}")
