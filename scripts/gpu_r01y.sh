#!/bin/bash
# Radix-sort scatter staged through shared memory: select/transpose/pagerank tests, C2 + C3 lines.
O=gpurun_out/${1:-r01y}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_transpose.py tests/test_gpu_pagerank.py tests/test_gpu_sampling.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 50 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1500 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
ls -la $O
