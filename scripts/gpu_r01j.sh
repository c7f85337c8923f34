#!/bin/bash
# Cold-row line split (TG_COLD_SPLIT_TAIL): GPU tests + C2 bench line.
O=gpurun_out/r01j; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
ls -la $O
