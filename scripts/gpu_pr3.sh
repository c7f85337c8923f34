#!/bin/bash
O=gpurun_out/${1:-r01z}; mkdir -p $O
for c in 148 74 296; do echo "== TG_SEG_CTAS=$c"; TG_SEG_CTAS=$c python scripts/seg_trace.py c2 2>&1 | grep segments; done > $O/seg_trace.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "rc=$?" >> $O/pytest_pr.log
for c in 148 74; do TG_SEG_CTAS=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench.err; done
