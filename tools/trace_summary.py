"""Print the top of a tools/trace_solve.py JSON file."""
import json
import sys

d = json.load(open(sys.argv[1]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
print({k: round(d[k], 2) if isinstance(d[k], float) else d[k]
       for k in ("iterations", "span_ms", "gpu_busy_ms", "idle_gaps_ms_total", "gaps_over_20us", "kernels")})
for t in d["top"][:n]:
    print(f"{t['total_ms']:8.2f} ms {t['count']:6d} x {t['avg_us']:8.1f} us  {t['name'][:70]}")
for g in d.get("gap_contexts", [])[:12]:
    print(f"  gap {g['total_ms']:7.2f} ms {g['count']:5d} x  {g['between']}")
