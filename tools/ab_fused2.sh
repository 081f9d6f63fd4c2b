#!/bin/bash
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" > gpurun_out/pytest_fused.log 2>&1
echo "tests: $(tail -1 gpurun_out/pytest_fused.log)"
grep -q " passed" gpurun_out/pytest_fused.log && ! grep -q failed gpurun_out/pytest_fused.log || { tail -60 gpurun_out/pytest_fused.log; exit 2; }
timeout -s KILL 300 python tools/micro/trace_head.py 256 > gpurun_out/trace_head2.txt 2>&1; tail -27 gpurun_out/trace_head2.txt
for v in 1 0; do
  export PCC_DEC_FUSED=$v
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
unset PCC_DEC_FUSED
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1; head -40 gpurun_out/launch_summary.txt
