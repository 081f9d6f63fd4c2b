#!/bin/bash
# ncu --set full of the longest launch of the hash / kernel-map / level kernels (the
# north_star's "achieved HBM GB/s for the gather/scatter and hash phases").
cd "$(dirname "$0")/.."
for k in "k_kmap:kmap" "k_hash_insert:hash_insert" "k_lvl_scatter:lvl_scatter" "k_expand:expand" "k_rs_hist:sort_hist"; do
  bash tools/ncu_biggest.sh "${k%%:*}" "full_${k##*:}"
done
