"""Per-kernel totals and shares from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("pcc::<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"^.*::", "", name)
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:40]:40s} {cnt[k]:8d} {v:10.1f} {100 * v / T:6.1f}%")
print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {T:10.1f}")
