#!/bin/bash
# Per-launch durations of the up/prune kernels (SIMT and tcgen05) + full captures of the largest.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
M=gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum
timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:k_up -c 40 --csv \
  --log-file gpurun_out/up_simt.csv python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
PCC_UP=tc timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:k_up -c 40 --csv \
  --log-file gpurun_out/up_tc.csv python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/up_simt.csv 2>&1 | tail -5
# largest launch index from the simt list
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_up -s ${S:-13} -c 1 \
  -o gpurun_out/full_up_simt python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
PCC_UP=tc timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:k_up -s ${S:-13} -c 1 \
  -o gpurun_out/full_up_tc python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
ls gpurun_out/
