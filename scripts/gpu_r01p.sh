#!/bin/bash
# K3: padded class-B windows; shared-memory carveout A/B.
O=gpurun_out/${1:-r01p}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest_pr.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pr.log
timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_pad.json 2> $O/bench_c2_pad.err
for c in 25 0; do
TIERGRAPH_PR_CARVEOUT=$c timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_carve$c.json 2> $O/bench_c2_carve$c.err
done
ls -la $O
