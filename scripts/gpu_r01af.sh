#!/bin/bash
# Sampler: offset wait moved to the member write; 256-word compaction blocks.
O=gpurun_out/${1:-r01af}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_gather.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 1500 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
ls -la $O
