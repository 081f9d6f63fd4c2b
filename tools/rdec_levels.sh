#!/bin/bash
# Per-level k_rans_dec durations of one B=256 cfg2 step under each PCC_RDEC setting (ncu launch list).
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
for e in "$@"; do
  env $e timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_rans_dec" -c 60 --csv \
    --log-file gpurun_out/rl.csv python tools/step_once.py --batch 256 --steps 0 > /dev/null 2>&1
  python - "$e" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/rl.csv")) if len(r) > 5]
h = rows[0]; iv = h.index("Metric Value")
t = [round(float(r[iv].replace(",", "")) / 1000) for r in rows[1:]]
print(sys.argv[1], sum(t), t)
PY
done
