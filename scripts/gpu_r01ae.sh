#!/bin/bash
# Parallel radix plan kernel: tests + C2 selection.
O=gpurun_out/${1:-r01ae}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_transpose.py tests/test_gpu_pagerank.py tests/test_gpu_sampling.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
ls -la $O
