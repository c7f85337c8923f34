#!/bin/bash
# K3 class-boundary sweep (TIERGRAPH_PR_LENA / _LENB), C2.
O=gpurun_out/${1:-r01x}; mkdir -p $O
for ab in 4096:512 2048:512 8192:512 4096:256 4096:1024 2048:256 8192:1024; do
  a=${ab%:*}; b=${ab#*:}
  TIERGRAPH_PR_LENA=$a TIERGRAPH_PR_LENB=$b timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 3 > $O/bench_c2_${a}_${b}.json 2> $O/bench_c2_${a}_${b}.err
done
ls -la $O
