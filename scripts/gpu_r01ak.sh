#!/bin/bash
# K1 grid: 1 / 2 / 4 CTAs per SM (fewer CTAs = fewer shared-memory flush atomics).
O=gpurun_out/${1:-r01ak}; mkdir -p $O
L=paper_2111_05894_b200/libtiergraph_b200.so
for v in indeg1 indeg2 indeg4; do
  cp variants/$v.so $L
  timeout 600 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu -k "degree" > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 3 > $O/bench_c2_$v.json 2> $O/bench_c2_$v.err
done
cp variants/indeg4.so $L
ls -la $O
