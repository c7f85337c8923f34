#!/bin/bash
# Round evidence: tests, smoke, C2 bench (default), launch list, per-kernel
# memory metrics (HBM / PCIe / NVLink) of every kernel, ncu --set full of K8
# and K3, and C3 / C4 bench lines. Usage: bash scripts/gpu_final.sh <tag>
set -x
O=gpurun_out/${1:-r01f}; mkdir -p $O
nvidia-smi -q -d CLOCK,POWER > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; free -g >> $O/lscpu.txt
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_c2_ref.json 2> $O/bench_c2_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sectors_aperture_sysmem_lookup_miss.sum,syslts__t_sectors_aperture_peer_lookup_miss.sum \
   --clock-control none --csv --log-file $O/kernel_memory.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_ncu_mem.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_bulk -s 5 -c 2 \
   -o $O/gather python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/ncu_gather.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pr_ -s 6 -c 2 \
   -o $O/prstep python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_pr.log 2>&1
timeout 1800 python bench.py --config c3 --steps 100 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gather_bulk -s 5 -c 2 \
   -o $O/gather_c3 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/ncu_gather_c3.log 2>&1
timeout 2400 python bench.py --config c4 --steps 100 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python -m pytest tests/test_distributed.py -x -q -m gpu > $O/pytest_distributed.log 2>&1; echo "rc=$?" >> $O/pytest_distributed.log
TG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c1 --steps 20 --warmup 3 > $O/bench_c1_2ranks_shared_gpu.json 2> $O/bench_c1_2ranks_shared_gpu.err
echo "rc=$?" >> $O/bench_c1_2ranks_shared_gpu.err
ls -la $O
