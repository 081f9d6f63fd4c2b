#!/bin/bash
# Round evidence: GPU tests, full default bench (JSON line), ncu launch list of one bench
# step, and ncu --set full captures of the dominant kernels (1 GPU).
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "gpu tests: $(tail -1 gpurun_out/pytest_gpu.log)"
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
tail -c 3000 gpurun_out/bench_default.log
# launch list of one timed step (skip the 3 warm-up steps' launches)
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 239 -c 239 --csv \
  --log-file gpurun_out/launches.csv python tools/step_once.py --batch 256 \
  > gpurun_out/ncu_launches.log 2>&1
echo "launch list: $(wc -l < gpurun_out/launches.csv) lines"
# full captures: decoder predictor at level 11 and the largest conv / up / rans_dec launches
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_head_tc -s 15 -c 1 \
  -o gpurun_out/full_head python tools/step_once.py --batch 256 > gpurun_out/ncu_full_head.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_rans_dec -s 15 -c 1 \
  -o gpurun_out/full_rdec python tools/step_once.py --batch 256 > gpurun_out/ncu_full_rdec.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_conv3_tc -s 8 -c 2 \
  -o gpurun_out/full_conv python tools/step_once.py --batch 256 > gpurun_out/ncu_full_conv.log 2>&1
ls -la gpurun_out/*.ncu-rep
