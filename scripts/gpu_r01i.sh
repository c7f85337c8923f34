#!/bin/bash
# Re-entry check after the container was re-created: GPU tests, smoke, the
# cold-row line-split probe, and the default C2 bench line.
O=gpurun_out/r01i; mkdir -p $O
timeout 300 python scripts/tail_probe.py > $O/tail_probe.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
ls -la $O
