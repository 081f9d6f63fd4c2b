#!/bin/bash
# End-of-session evidence: full GPU test suite, the workload sweep, then the profile round.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1
echo "gpu tests: $(tail -1 gpurun_out/pytest_gpu_final.log)"
bash tools/sweep_r02.sh
bash tools/profile_round.sh
