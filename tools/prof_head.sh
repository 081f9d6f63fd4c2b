cd $GRAFT_REPO_ROOT
bash tools/ncu_biggest.sh "k_head_tc<.int.32, .int.32, .int.1" head_dec
ncu -i gpurun_out/head_dec.ncu-rep --page raw --csv > gpurun_out/head_dec_raw.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/head_dec.ncu-rep 60 > gpurun_out/head_dec_hot.txt 2>&1
timeout -s KILL 300 python tools/micro/trace_head.py 256 > gpurun_out/trace_head.txt 2>&1
