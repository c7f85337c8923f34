#!/bin/bash
# K8 rows per warp batch at C3 (first round spreads cold rows over more warps).
O=gpurun_out/${1:-r01aa}; mkdir -p $O
for b in 4 8 32; do
  TIERGRAPH_GATHER_ROWS_PER_WARP=$b timeout 1500 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c3_b$b.json 2> $O/bench_c3_b$b.err
done
for b in 4 8 32; do
  TIERGRAPH_GATHER_ROWS_PER_WARP=$b timeout 600 python bench.py --steps 50 --no-cpu-baseline > $O/bench_c2_b$b.json 2> $O/bench_c2_b$b.err
done
ls -la $O
