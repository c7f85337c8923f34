#!/bin/bash
O=gpurun_out/r01c4a; mkdir -p $O
free -g > $O/free.txt
timeout 1200 python scripts/alias_probe.py ${1:-8} > $O/alias_probe.log 2>&1; echo "rc=$?" >> $O/alias_probe.log
free -g >> $O/free.txt
