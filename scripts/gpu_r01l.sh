#!/bin/bash
# K8 dynamic batch claims (TG_GATHER_DYNAMIC) A/B at C2 and C3 + gather tests.
O=gpurun_out/r01l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gather.py -x -q -m gpu > $O/pytest_gather.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gather.log
for m in bulk+spread bulk+spread+dynamic; do
  timeout 600 python bench.py --no-cpu-baseline --gather-mode $m > $O/bench_c2_$m.json 2> $O/bench_c2_$m.err
done
for m in bulk+spread bulk+spread+dynamic; do
  timeout 900 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline --gather-mode $m > $O/bench_c3_$m.json 2> $O/bench_c3_$m.err
done
ls -la $O
