#!/bin/bash
O=gpurun_out/${1:-r01c3pr}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_gather.py -x -q -m gpu > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1800 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
