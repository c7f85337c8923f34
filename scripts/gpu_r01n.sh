#!/bin/bash
# K3 hot columns A/B: PageRank tests + C2 bench with and without.
O=gpurun_out/${1:-r01n}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pr.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2_hot.json 2> $O/bench_c2_hot.err
TIERGRAPH_PR_HOT_COLUMNS=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2_nohot.json 2> $O/bench_c2_nohot.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_ncu.log 2>&1
ls -la $O
