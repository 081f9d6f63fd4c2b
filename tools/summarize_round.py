"""Turn the gpurun_out/ outputs of tools/profile_round.sh into the tracked profiles/ files.

usage: python tools/summarize_round.py r01
  profiles/<tag>_bench.json         the default bench.py JSON line
  profiles/<tag>_bench_reference.json  the --impl reference line
  profiles/<tag>_launches.txt       per-kernel totals / shares of one B=512 step (ncu launch list)
  profiles/<tag>_ncu_full_<k>.txt   key metrics + DRAM bytes of the longest launch of kernel k
  profiles/traffic.json             DRAM bytes of those launches (bench.py roofline.traffic)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
KEYS = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Warp Cycles Per Issued Instruction", "Executed Instructions"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__inst_executed_pipe_alu",
       "sm__inst_executed_pipe_fma", "sm__inst_executed_pipe_lsu", "sm__pipe_tensor_cycles_active",
       "smsp__inst_executed_op_utcimma", "sm__inst_executed_pipe_uniform"]


def ncu_csv(path, page):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, u):
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def summarize(tag, name, path):
    rows = ncu_csv(path, "details")
    hdr = rows[0]
    m = {r[hdr.index("Metric Name")]: (r[hdr.index("Metric Value")], r[hdr.index("Metric Unit")]) for r in rows[1:]}
    kname = rows[1][hdr.index("Kernel Name")] if len(rows) > 1 else "?"
    raw = ncu_csv(path, "raw")
    rh, ru, rv = raw[0], raw[1], raw[2]
    lines = [f"== {name}: longest launch of one B=512 step (ncu --set full --clock-control none)",
             f"   kernel: {kname[:110]}"]
    for k in KEYS:
        if k in m:
            lines.append(f"   {k:40s} {m[k][0]} {m[k][1]}")
    dram = 0.0
    for j, h in enumerate(rh):
        if any(h.startswith(p) for p in RAW) and (h.endswith(".sum") or "pct_of_peak_sustained_active" in h):
            if h.startswith("sm__inst_executed_pipe") and not h.endswith("avg.pct_of_peak_sustained_active"):
                continue
            if h.startswith("sm__pipe_tensor") and not h.endswith("avg.pct_of_peak_sustained_active"):
                continue
            lines.append(f"   {h:60s} {rv[j]} {ru[j]}")
        if h in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram += to_bytes(rv[j], ru[j])
    open(os.path.join(PROF, f"{tag}_ncu_full_{name}.txt"), "w").write("\n".join(lines) + "\n")
    return dram, m.get("Duration")


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    for src, dst in (("bench_default.log", "bench.json"), ("bench_reference.log", "bench_reference.json")):
        p = os.path.join(OUT, src)
        if os.path.exists(p):
            line = [l for l in open(p).read().splitlines() if l.startswith("{")][-1]
            open(os.path.join(PROF, f"{tag}_{dst}"), "w").write(json.dumps(json.loads(line), indent=1) + "\n")
    p = os.path.join(OUT, "launches.csv")
    if os.path.exists(p):
        s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), p],
                           capture_output=True, text=True).stdout
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write(
            "# ncu --metrics gpu__time_duration.sum --clock-control none, one B=512 cfg2 step (one bench lane) through one codec\n"
            "# instance (tools/step_once.py --batch 512 --steps 0): cold-cache, serialised launches\n" + s)
    traffic = {}
    for f in sorted(os.listdir(OUT)):
        if f.startswith("full_") and f.endswith(".ncu-rep"):
            name = f[5:-8]
            dram, dur = summarize(tag, name, os.path.join(OUT, f))
            traffic[name] = {"dram_bytes_per_launch": dram, "launch": "longest launch of one B=512 step",
                             "duration": " ".join(dur) if dur else None, "source": f"profiles/{tag}_ncu_full_{name}.txt"}
    if traffic:  # keyed by workload (bench.py measured_traffic): these captures are cfg2 steps
        p = os.path.join(PROF, "traffic.json")
        try:
            old = json.load(open(p))
            old = old if all(isinstance(v, dict) and "dram_bytes_per_launch" not in v for v in old.values()) else {}
        except Exception:
            old = {}
        old["cfg2"] = traffic
        json.dump(old, open(p, "w"), indent=1)
    for t in ("memcheck", "racecheck", "synccheck"):
        p = os.path.join(OUT, f"sanitize_{t}.txt")
        if os.path.exists(p):
            keep = [l for l in open(p).read().splitlines()
                    if l.startswith("ok ") or "SUMMARY" in l or "Error" in l or "ERROR" in l or "Hazard" in l]
            open(os.path.join(PROF, f"{tag}_sanitize_{t}.txt"), "w").write(
                f"# compute-sanitizer --tool {t} python tools/sanitize_cfg1.py (cfg1 frame; C = 8 / 32; "
                "XFP-off, GRED-off and raw-freq models)\n" + "\n".join(keep) + "\n")
    print("wrote", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
