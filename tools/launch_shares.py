"""Kernel shares of an ncu launch list (`--metrics gpu__time_duration.sum --csv`) as a markdown table.

    python tools/launch_shares.py profiles/r02_launches_cfg5.csv "title" > profiles/r02_launches_cfg5.md
"""
import collections
import csv
import sys

path, title = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = next(r for r in rows if "Kernel Name" in r)
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows:
    if len(r) != len(hdr) or r is hdr or r[vi] == "Metric Value":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    us = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v / 1e3)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
n = sum(a[0] for a in agg.values())
print(f"# {title}\n")
print(f"Serialised kernel time: {tot / 1e3:.1f} ms over {n} launches (ncu serialises launches and runs each with a cold "
      "L2; the shares, not the absolute times, compare with the event-timed run).\n")
print("| kernel | launches | ms | share |\n|---|---|---|---|")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    if a[1] / tot < 0.0005:
        continue
    print(f"| `{name[:90]}` | {a[0]} | {a[1] / 1e3:.2f} | {100 * a[1] / tot:.1f} % |")
