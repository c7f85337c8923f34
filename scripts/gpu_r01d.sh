set -x
O=gpurun_out/r01d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_select.py -q -x > $O/pytest_pr.log 2>&1; echo rc=$? >> $O/pytest_pr.log
timeout 600 python scripts/pr_probe.py c2 > $O/pr_probe.log 2>&1
