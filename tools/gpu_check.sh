#!/bin/bash
# GPU round trip used during development: build, parity tests (hard-killed on hang), bench.
# usage: tools/gpu_check.sh [batch sizes...]
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -x -q -k "per_tensor and 32" > gpurun_out/pytest_quick.log 2>&1
echo "quick: $(tail -1 gpurun_out/pytest_quick.log)"
grep -q passed gpurun_out/pytest_quick.log || exit 2
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "gpu tests: $(tail -1 gpurun_out/pytest_gpu.log)"
for b in "${@:-256}"; do
  timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --batch $b --no-cpu-baseline > gpurun_out/bench_b$b.log 2>&1
  python - "$b" <<'PY'
import json, sys
b = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_b{b}.log").read().strip().splitlines()[-1])
    print(b, round(d["value"]), round(d["enc_fps"]), round(d["dec_fps"]), d["profile_ms_per_step"])
except Exception as e:
    print("bench failed", b, e)
    print(open(f"gpurun_out/bench_b{b}.log").read()[-2000:])
PY
done
