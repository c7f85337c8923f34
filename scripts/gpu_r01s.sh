#!/bin/bash
# Sampler lanes: sampling tests + C2 bench (lanes 4 vs 1).
O=gpurun_out/${1:-r01s}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_gather.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_l4.json 2> $O/bench_c2_l4.err
TIERGRAPH_SAMPLER_LANES=1 timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_l1.json 2> $O/bench_c2_l1.err
TIERGRAPH_SAMPLER_LANES=8 timeout 600 python bench.py --no-cpu-baseline --steps 50 > $O/bench_c2_l8.json 2> $O/bench_c2_l8.err
ls -la $O
