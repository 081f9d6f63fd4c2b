#!/bin/bash
# A/B of environment overrides on the bench: tools/ab_env.sh "VAR=a" "VAR=b" ...
cd "$(dirname "$0")/.."
python paper_2603_25260_b200/build.py > /dev/null || exit 1
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ab_$i.log 2>&1
  python - "$i" "$e" <<'PY'
import json, sys
i, e = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/bench_ab_{i}.log").read().strip().splitlines()[-1])
    p = d["profile_ms_per_step"]
    print(e, round(d["value"]), round(d["enc_fps"]), round(d["dec_fps"]), d["parity_sample_frame0"], {k: p[k] for k in ("sort", "scan", "octree", "morton", "head_dec", "head_enc", "conv", "up")})
except Exception as ex:
    print("bench failed", e, ex); print(open(f"gpurun_out/bench_ab_{i}.log").read()[-1500:])
PY
done
