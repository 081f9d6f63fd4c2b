"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = [line]
        blocks.append(cur)
    elif cur is not None:
        cur.append(line)
for b in blocks:
    rows = list(csv.reader(b))
    print("==", rows[0][1][:90])
    hdr = rows[1]
    si, ki = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[ki]), r[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(v for v, _ in data) or 1
    for v, s in sorted(data, reverse=True)[:n]:
        print(f"  {100 * v / tot:5.1f}%  {s[:100]}")
