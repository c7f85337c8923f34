#!/bin/bash
# K3 register caps A/B (library variants swapped in place): hub 80 regs; + class B/C 64 regs.
O=gpurun_out/${1:-r01u}; mkdir -p $O
L=paper_2111_05894_b200/libtiergraph_b200.so
for v in hub80 hub80_step64; do
  cp variants/$v.so $L
  timeout 600 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest_pr_$v.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pr_$v.log
  timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_$v.json 2> $O/bench_c2_$v.err
done
ls -la $O
