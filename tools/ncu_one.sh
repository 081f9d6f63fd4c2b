#!/bin/bash
# usage: [ENV=..] tools/ncu_one.sh KERNEL_REGEX SKIP NAME  -> gpurun_out/NAME.ncu-rep (one launch, --set full)
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:$1 -s $2 -c 1 \
  -o gpurun_out/$3 python tools/step_once.py --batch 512 --steps 0 > gpurun_out/$3.log 2>&1
tail -3 gpurun_out/$3.log
