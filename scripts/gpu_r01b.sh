set -x
O=gpurun_out/r01b; mkdir -p $O
timeout 1200 python -m pytest tests/test_dropin.py -q -m gpu -x > $O/pytest_dropin.log 2>&1; echo rc=$? >> $O/pytest_dropin.log
for c in 1 2 3 4 6 7 8 9; do timeout 300 oracle/_ref/dropin/acceptance_b200 $c; done > $O/acceptance_b200.log 2>&1
timeout 300 oracle/_ref/dropin/unit_b200 > $O/unit_b200.log 2>&1
timeout 300 python scripts/pcie_probe.py > $O/pcie_probe.log 2>&1
timeout 600 python scripts/gather_modes.py c2 > $O/gather_modes.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
