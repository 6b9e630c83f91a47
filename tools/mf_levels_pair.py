"""Pair the rows of tools/mf_levels.py with the solve launches of an ncu
launch list of the same process (--metrics gpu__time_duration.sum --csv,
-k regex:mf_): the last len(rows) launches of the solve kernels.

    python tools/mf_levels_pair.py rows.json launches.csv
"""
import csv
import json
import sys

rows = json.loads([l for l in open(sys.argv[1]) if l.startswith("[")][-1])
cs = list(csv.reader(open(sys.argv[2])))
hi = [i for i, r in enumerate(cs) if "Kernel Name" in r][0]
h = cs[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
L = []
for r in cs[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki]
    if not any(k in name for k in ("mf_gather_kernel", "mf_rows_kernel", "mf_merged_kernel")):
        continue
    L.append((name.split("(")[0], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)))
L = L[-len(rows):]
assert len(L) == len(rows), (len(L), len(rows))
tot = sum(t for _, t in L)
print(f"total {tot:.1f} us over {len(L)} launches; "
      f"{sum(r['bytes'] for r in rows) / 1e9:.2f} GB")
print("level phase    time_us        MB     GB/s  fronts  p_avg  b_avg")
for r, (name, t) in zip(rows, L):
    extra = (f"{r['fronts']:7d} {r['p_avg']:6.0f} {r['b_avg']:6.0f}" if "fronts" in r else "")
    print(f"L{r['level']:2d} {r['phase']:7s} {t:8.1f} {r['bytes'] / 1e6:9.1f} "
          f"{r['bytes'] / t / 1e3:8.0f} {extra}")
