#!/bin/bash
# Dev loop on one GPU: build, a pytest selection ($1, -k expression), the default bench
# line (5 steps) and optional extra bench workloads ($2.., e.g. cfg3).
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ -n "$1" ]; then
  timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_quick.log 2>&1
  echo "tests: $(tail -1 gpurun_out/pytest_quick.log)"
  grep -q " passed" gpurun_out/pytest_quick.log && ! grep -q "failed" gpurun_out/pytest_quick.log || { tail -60 gpurun_out/pytest_quick.log; exit 2; }
fi
shift
for w in cfg2 "$@"; do
  timeout -s KILL 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-latency > gpurun_out/bench_q_$w.log 2>&1
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_q_{w}.log").read().strip().splitlines()[-1])
    p = d["profile_ms_per_step"]
    print(w, round(d["value"]), "enc", round(d.get("enc_fps") or 0), "dec", round(d.get("dec_fps") or 0), "parity", d["parity"]["ok"],
          sorted(((k, round(v, 2)) for k, v in p.items()), key=lambda x: -x[1])[:9])
except Exception as ex:
    print("bench failed", w, ex); print(open(f"gpurun_out/bench_q_{w}.log").read()[-1500:])
PY
done
