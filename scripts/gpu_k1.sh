#!/bin/bash
O=gpurun_out/${1:-r01k1}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "rc=$?" >> $O/pytest_pr.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
