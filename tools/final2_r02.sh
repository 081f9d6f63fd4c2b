#!/bin/bash
# Evidence at the 2048-frame default: launch-configuration tests, sweep of the L <= 12
# workloads (bench defaults), then the profile round.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 1200 python -m pytest tests -m gpu -q -k "launch_configuration" > gpurun_out/pytest_lc.log 2>&1
echo "launch-configuration tests: $(tail -1 gpurun_out/pytest_lc.log)"
out=gpurun_out/sweep2_r02.jsonl
: > $out
for w in cfg2 cfg1 cfg2_L11 cfg2_t3 cfg2_xfp_off cfg2_gred_off cfg2_rawfreq; do
  timeout -s KILL 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep2_$w.log 2>&1
  tail -1 gpurun_out/sweep2_$w.log | grep '^{' >> $out || echo "{\"workload_failed\": \"$w\"}" >> $out
  echo "$w done"
done
bash tools/profile_round.sh
