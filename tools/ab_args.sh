#!/bin/bash
# bench.py argument A/B: tools/ab_args.sh "--streams 4" "--streams 4 --pipeline" ...
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
for a in "$@"; do
  timeout -s KILL 400 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-latency > gpurun_out/bench_a.log 2>&1
  python - "$a" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/bench_a.log").read().strip().splitlines()[-1])
    print(sys.argv[1], "|", round(d["value"]), "enc", round(d["enc_fps"]), "dec", round(d["dec_fps"]), "e2e", round(d["e2e"]["value"]), "parity", d["parity"]["ok"], "ms", round(d["ms_per_step"], 2))
except Exception as ex:
    print("bench failed", sys.argv[1], ex); print(open("gpurun_out/bench_a.log").read()[-1500:])
PY
done
