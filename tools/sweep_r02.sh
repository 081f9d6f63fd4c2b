#!/bin/bash
# Bench lines of every workload (BASELINE configs + NEXT-1/NEXT-4 variants) at HEAD.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
out=gpurun_out/sweep_r02.jsonl
: > $out
for w in cfg2 cfg1 cfg3 cfg5 cfg2_L11 cfg2_L13 cfg2_L14 cfg2_L15 cfg2_L16 cfg2_t3 cfg2_xfp_off cfg2_gred_off cfg2_rawfreq; do
  timeout -s KILL 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$w.log 2>&1
  tail -1 gpurun_out/sweep_$w.log | grep '^{' >> $out || echo "{\"workload_failed\": \"$w\"}" >> $out
  echo "$w done"
done
