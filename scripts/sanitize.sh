#!/bin/bash
# compute-sanitizer over the small-input driver (scripts/sanitize_driver.py):
# memcheck, racecheck, synccheck and initcheck on every case; logs under $1.
O=${1:-gpurun_out/sanitize}; mkdir -p $O
export TG_UNDER_SANITIZER=1 PYTHONUNBUFFERED=1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for c in k8 k8ldg k1 sampler k3 mgraph select transpose peers; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    # check only this library's kernels (namespace tgb), not torch's -- except
    # under initcheck, which must see torch's fills (zeroed flags) as writes
    filt="--kernel-name kns=3tgb"
    [ $tool = initcheck ] && filt=""
    timeout 1500 $CS --tool $tool $extra --print-limit 200 $filt \
      python scripts/sanitize_driver.py $c > $O/sanitize_${tool}_$c.log 2>&1
    echo "rc=$?" >> $O/sanitize_${tool}_$c.log
  done
done
grep -H -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize case|rc=" $O/sanitize_*.log > $O/sanitize_summary.txt
