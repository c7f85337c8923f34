set -x
O=gpurun_out/r01c; mkdir -p $O
./scripts/micro/dadd_chain > $O/dadd_chain.log 2>&1
timeout 600 python scripts/pr_probe.py c2 > $O/pr_probe.log 2>&1
timeout 600 python scripts/gather_modes.py c2 > $O/gather_modes.log 2>&1
