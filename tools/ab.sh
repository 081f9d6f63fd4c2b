#!/bin/bash
# A/B of environment overrides on one bench workload: tools/ab.sh WORKLOAD "VAR=a" "VAR=b" ...
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
w=$1; shift
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout -s KILL 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-latency > gpurun_out/bench_ab_$i.log 2>&1
  python - "$i" "$e" <<'PY'
import json, sys
i, e = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/bench_ab_{i}.log").read().strip().splitlines()[-1])
    p = d["profile_ms_per_step"]
    print(e, round(d["value"]), "enc", round(d.get("enc_fps") or 0), "dec", round(d.get("dec_fps") or 0), "parity", d["parity"]["ok"],
          sorted(((k, round(v, 2)) for k, v in p.items()), key=lambda x: -x[1])[:8])
except Exception as ex:
    print("bench failed", e, ex); print(open(f"gpurun_out/bench_ab_{i}.log").read()[-1500:])
PY
done
