#!/bin/bash
# K3: class-B/C target loads skip L1.
O=gpurun_out/${1:-r01q}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pr.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_$i.json 2> $O/bench_c2_$i.err; done
ls -la $O
