#!/bin/bash
# usage: [ENV=..] tools/ncu_biggest.sh KERNEL_REGEX NAME [MAXLAUNCHES]
# launch list of the kernel over one B=256 step, then --set full of its longest launch.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k "regex:$1" -c ${3:-60} --csv \
  --log-file gpurun_out/$2_list.csv python tools/step_once.py --batch 512 --steps 0 > /dev/null 2>&1
IDX=$(python - "$2" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_list.csv")) if len(r) > 5]
h = rows[0]
t = [(float(r[h.index("Metric Value")].replace(",", "")), i) for i, r in enumerate(rows[1:])]
print(max(t)[1])
PY
)
echo "longest launch index $IDX"
timeout -s KILL 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$1" -s $IDX -c 1 \
  -o gpurun_out/$2 python tools/step_once.py --batch 512 --steps 0 > gpurun_out/$2.log 2>&1
tail -2 gpurun_out/$2.log
