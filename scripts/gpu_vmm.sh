#!/bin/bash
# host-page translation experiment (VMM host allocation vs cudaHostAlloc vs THP)
O=gpurun_out/r01v; mkdir -p $O
{ cat /sys/kernel/mm/transparent_hugepage/enabled; cat /sys/kernel/mm/transparent_hugepage/defrag; nproc; free -g; numactl -H 2>/dev/null | head -3; } > $O/sys.txt 2>&1
timeout 600 scripts/micro/host_vmm 57 VAB > $O/host_vmm.log 2>&1
echo "rc=$?" >> $O/host_vmm.log
# multi-process path on one GPU (gloo plumbing, CUDA-IPC peers)
TG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c1 --steps 20 --warmup 3 > $O/bench_share2.json 2> $O/bench_share2.err
echo "rc=$?" >> $O/bench_share2.err
