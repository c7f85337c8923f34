#!/bin/bash
# K3 check: pagerank parity tests + a short C2 bench (PageRank sub-object) + ncu of K3
O=gpurun_out/${1:-r01x}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_distributed.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "rc=$?" >> $O/pytest_pr.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pr_ -s 9 -c 3 -o $O/prstep python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_pr.log 2>&1
