#!/bin/bash
# bench.py lane-count / batch A/B: tools/ab_streams.sh "S B" ...
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
for sb in "$@"; do
  set -- $sb
  timeout -s KILL 400 python bench.py --streams $1 --batch $2 --steps 5 --warmup 3 --no-cpu-baseline --no-latency --no-parity > gpurun_out/bench_s.log 2>&1
  python - "$sb" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/bench_s.log").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]), "enc", round(d["enc_fps"]), "dec", round(d["dec_fps"]), "e2e", round(d["e2e"]["value"]))
except Exception as ex:
    print("bench failed", sys.argv[1], ex); print(open("gpurun_out/bench_s.log").read()[-800:])
PY
done
