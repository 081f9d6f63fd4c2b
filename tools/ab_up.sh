#!/bin/bash
# A/B of the up/prune kernels: parity with the tcgen05 variant forced, then bench both.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "gpu tests: $(tail -1 gpurun_out/pytest_gpu.log)"
grep -q " passed" gpurun_out/pytest_gpu.log || { tail -60 gpurun_out/pytest_gpu.log; exit 2; }
PCC_UP=tc timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -x -q -k "per_tensor or batch_bitstream" > gpurun_out/pytest_uptc.log 2>&1
echo "uptc tests: $(tail -1 gpurun_out/pytest_uptc.log)"
grep -q " passed" gpurun_out/pytest_uptc.log || { tail -60 gpurun_out/pytest_uptc.log; exit 2; }
for v in tc simt; do
  PCC_UP=$v timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_up_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/bench_up_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']),d.get('profile_ms_per_step'))"
done
