#!/bin/bash
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "gpu tests: $(tail -1 gpurun_out/pytest_gpu.log)"
grep -q " passed" gpurun_out/pytest_gpu.log || { tail -60 gpurun_out/pytest_gpu.log; exit 2; }
M=gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:k_up -c 28 --csv \
  --log-file gpurun_out/up_tc4.csv python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_up -s 13 -c 1 \
  -o gpurun_out/full_up_tc4 python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
ls gpurun_out | tail -3
