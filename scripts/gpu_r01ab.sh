#!/bin/bash
# Radix scatter at <= 80 registers (3 CTAs per SM): tests + C2/C3 selection.
O=gpurun_out/${1:-r01ab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_transpose.py tests/test_gpu_pagerank.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1500 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
ls -la $O
