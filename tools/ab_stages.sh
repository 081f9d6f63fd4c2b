#!/bin/bash
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "batch_bitstream or decoder or multi_segment" > gpurun_out/pytest_st.log 2>&1
echo "tests: $(tail -1 gpurun_out/pytest_st.log)"
for v in auto 2 3 4; do
  if [ $v = auto ]; then unset PCC_DEC_STAGES; else export PCC_DEC_STAGES=$v; fi
  timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_st_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/bench_st_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']),d['profile_ms_per_step']['rans_dec'])"
done
