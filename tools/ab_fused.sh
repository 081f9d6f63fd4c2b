#!/bin/bash
# fused decoder: parity (forced on / off) and bench A/B (auto, forced off, forced on)
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or batch or errors or large" > gpurun_out/pytest_fused.log 2>&1
echo "tests: $(tail -1 gpurun_out/pytest_fused.log)"
grep -q " passed" gpurun_out/pytest_fused.log && ! grep -q failed gpurun_out/pytest_fused.log || { tail -60 gpurun_out/pytest_fused.log; exit 2; }
for v in auto 0 1; do
  if [ $v = auto ]; then unset PCC_DEC_FUSED; else export PCC_DEC_FUSED=$v; fi
  timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fused_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_fused_{v}.log").read().strip().splitlines()[-1])
    print(v, round(d["value"]), round(d["enc_fps"]), round(d["dec_fps"]), d["parity_sample_frame0"], d["profile_ms_per_step"])
except Exception as e:
    print("bench failed", v, e); print(open(f"gpurun_out/bench_fused_{v}.log").read()[-2000:])
PY
done
