"""Top SASS lines by executed instructions (ncu --page source --print-source sass)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
si, ii, wi = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for idx, r in enumerate(rows[1:]):
    try:
        data.append((float(r[ii]), float(r[wi]), idx, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
totw = sum(d[1] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
# instructions by address region: print cumulative executed per contiguous block of 50 lines
blk = {}
for e, w, idx, s in data:
    blk.setdefault(idx // 50, [0, 0])
    blk[idx // 50][0] += e
    blk[idx // 50][1] += w
print("block(50 lines)  %instr  %stall")
for b, (e, w) in sorted(blk.items()):
    if e / tot > 0.01 or w / totw > 0.01:
        print(f"  {b * 50:5d}-{b * 50 + 49:5d}  {100 * e / tot:5.1f}  {100 * w / totw:5.1f}")
