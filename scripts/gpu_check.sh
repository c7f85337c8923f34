#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full captures.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
set -x
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi -q -d CLOCK,POWER > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; free -g >> $O/lscpu.txt
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather -s 5 -c 2 \
   -o $O/gather python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/ncu_gather.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pr_ -s 6 -c 2 \
   -o $O/prstep python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_pr.log 2>&1
ls -la $O
