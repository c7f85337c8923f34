#!/bin/bash
# One-pass ncu DRAM/sysmem traffic of K8 at C3 and C4 (no kernel replay, so
# no device-memory save/restore of the 57 GB / 86 GB working sets).
O=gpurun_out/${1:-r01v}; mkdir -p $O
for c in c3 c4; do
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__t_sectors_aperture_sysmem_lookup_miss.sum \
   --clock-control none --csv --log-file $O/k8_traffic_$c.csv -k regex:gather_bulk -s 3 -c 5 \
   python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/ncu_traffic_$c.log 2>&1
done
ls -la $O
