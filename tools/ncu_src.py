"""Per-CUDA-source-line instruction counts and stall samples of one kernel in
an ncu report (ncu --page source --print-source cuda,sass).

    python tools/ncu_src.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = "", None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    num = lambda v: int(v) if v.strip().isdigit() else 0
    ws, ie = num(r[4]), num(r[7])
    agg.append((ws, ie, f"{fname}:{r[0]}  {r[1].strip()[:90]}"))
tot_s = sum(a[0] for a in agg) or 1
tot_i = sum(a[1] for a in agg) or 1
print(f"samples {tot_s}, warp instructions {tot_i}")
for ws, ie, k in sorted(agg, key=lambda a: -a[0])[:top]:
    print(f"{100 * ws / tot_s:5.1f}% smp {100 * ie / tot_i:5.1f}% ins  {k}")
