#!/bin/bash
# K3 class-B lanes per row (4 / 8 / 16), library variants swapped in place.
O=gpurun_out/${1:-r01aj}; mkdir -p $O
L=paper_2111_05894_b200/libtiergraph_b200.so
for v in blanes4 blanes8 blanes16; do
  cp variants/$v.so $L
  timeout 600 python -m pytest tests/test_gpu_pagerank.py tests/test_golden.py -x -q -m gpu > $O/pytest_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_$v.log
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 3 > $O/bench_c2_$v.json 2> $O/bench_c2_$v.err
done
cp variants/blanes8.so $L
ls -la $O
