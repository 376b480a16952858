"""Per-kernel totals of an ncu launch list (``ncu --metrics gpu__time_duration.sum
--csv --log-file launches.csv ...``): count, total ms, share, average us.

    python tools/ncu_launch_summary.py launches.csv [top]
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
hdr = rows[0]
ik, im, iv, iu = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[r[iu]]
    name = re.sub(r"\(.*$", "", r[ik]).replace("void ", "")
    tot[name] += v
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"{'kernel':64s} {'n':>6s} {'total_ms':>9s} {'share':>6s} {'avg_us':>9s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{k[:64]:64s} {cnt[k]:6d} {v:9.3f} {100 * v / all_ms:5.1f}% {1e3 * v / cnt[k]:9.2f}")
print(f"{'TOTAL':64s} {sum(cnt.values()):6d} {all_ms:9.3f}")
