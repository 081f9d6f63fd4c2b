cd $GRAFT_REPO_ROOT
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "octree or batch or large or errors" 2>&1 | tail -2
bash tools/ab_env.sh PCC_SORT_DB=8 PCC_SORT_DB=9
