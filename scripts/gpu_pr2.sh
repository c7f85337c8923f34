#!/bin/bash
O=gpurun_out/${1:-r01y}; mkdir -p $O
python scripts/seg_trace.py c2 > $O/seg_trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_distributed.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "rc=$?" >> $O/pytest_pr.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
