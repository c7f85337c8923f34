#!/bin/bash
O=gpurun_out/r01w; mkdir -p $O
timeout 600 python -m pytest tests/test_distributed.py -x -q -m gpu > $O/pytest_ipc.log 2>&1; echo "rc=$?" >> $O/pytest_ipc.log
TG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c1 --steps 20 --warmup 3 > $O/bench_share2.json 2> $O/bench_share2.err
echo "rc=$?" >> $O/bench_share2.err
