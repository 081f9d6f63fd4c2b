#!/bin/bash
# Round evidence on one GPU: the default bench line, the reference arm, the ncu launch
# list of one B=256 cfg2 step and ncu --set full of the longest launch of each hot kernel.  Outputs land in gpurun_out/; tools/summarize_round.py
# turns them into profiles/.
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
tail -c 300 gpurun_out/bench_default.log
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1
tail -c 300 gpurun_out/bench_reference.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/step_once.py --batch 512 --steps 0 > gpurun_out/ncu_launches.log 2>&1
echo "launch list: $(wc -l < gpurun_out/launches.csv) lines"
for k in "k_head4_tc<.int.32, .int.32, .int.1:head_dec" "k_head4_tc<.int.32, .int.32, .int.0:head_enc" \
         "k_rans_dec_t:rans_dec" "k_conv3_ws:conv" "k_up_tc:up" "k_down_tc:down" "k_rs_scatter:sort_scatter" \
         "k_morton_dedup:morton" "k_kmap_derive:kmap" "k_rans_enc:rans_enc"; do
  bash tools/ncu_biggest.sh "${k%%:*}" "full_${k##*:}"
done
# compute-sanitizer is closed on this pool (runs under it left GPUs needing a reset)
ls gpurun_out/*.ncu-rep
