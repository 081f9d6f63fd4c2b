#!/bin/bash
# NEXT-row measurements on one GPU: HRCS report, precision sweep / t = L-3 bench lines,
# cfg3 bench line, float twin cross-device test.  Outputs land in gpurun_out/.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 600 python tools/hrcs_report.py --frames 64 > gpurun_out/hrcs.txt 2>&1
tail -3 gpurun_out/hrcs.txt
for w in cfg2_L11 cfg2_L12 cfg2_L13 cfg2_L14 cfg2_L15 cfg2_L16 cfg2_t3 cfg3; do
  timeout -s KILL 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1
  tail -1 gpurun_out/bench_$w.log | cut -c1-200
done
timeout -s KILL 300 python -m pytest tests/test_float_twin.py -q -s -m gpu > gpurun_out/float_twin_gpu.log 2>&1
grep "float twin" gpurun_out/float_twin_gpu.log
