#!/bin/bash
O=gpurun_out/r01c4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q -m gpu > $O/pytest_gather.log 2>&1; echo "rc=$?" >> $O/pytest_gather.log
( while true; do free -g | sed -n 2p; nvidia-smi --query-gpu=memory.used --format=csv,noheader; sleep 20; done ) > $O/mem_trace.txt 2>&1 &
MON=$!
timeout 2400 python bench.py --config c4 --steps 50 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
echo "rc=$?" >> $O/bench_c4.err
kill $MON
