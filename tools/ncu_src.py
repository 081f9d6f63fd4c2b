"""Per-opcode and per-stall-reason breakdown of an ncu --set full --import-source report
(source page, SASS): python tools/ncu_src.py REPORT [top_lines]."""
import csv
import subprocess
import sys
from collections import Counter


def main(path, top=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    ia, isrc, iex, ismp = (h.index("Address"), h.index("Source"), h.index("Instructions Executed"),
                           h.index("Warp Stall Sampling (All Samples)"))
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or c.startswith("Warp Stall Sampling (All Samples) -")]
    data = [r for r in rows[2:] if len(r) > iex]
    tot = sum(int(r[iex] or 0) for r in data)
    smp = sum(int(r[ismp] or 0) for r in data)
    print(f"instructions {tot}, stall samples {smp}")
    c, cs = Counter(), Counter()
    for r in data:
        s = r[isrc].split()
        op = (s[1] if s and s[0].startswith("@") else (s[0] if s else "?")).split(".")[0]
        c[op] += int(r[iex] or 0)
        cs[op] += int(r[ismp] or 0)
    for k, v in c.most_common(22):
        print(f"  {k:10s} {100 * v / tot:6.2f}% instr {100 * cs[k] / max(smp, 1):6.2f}% samples")
    if top:
        print("hottest lines (stall samples):")
        for r in sorted(data, key=lambda r: -int(r[ismp] or 0))[:top]:
            print(f"  {int(r[ismp] or 0):6d} {int(r[iex] or 0):10d}  {r[isrc][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
