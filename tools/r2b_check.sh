#!/bin/bash
# Session check at HEAD: GPU tests, default bench line, cfg3 line.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "gpu tests: $(tail -1 gpurun_out/pytest_gpu.log)"
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1
tail -c 400 gpurun_out/bench_default.log; echo
timeout -s KILL 600 python bench.py --workload cfg3 --steps 5 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1
tail -c 300 gpurun_out/bench_cfg3.log; echo
