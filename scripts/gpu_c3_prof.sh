# ncu of K8 and K3 at C3 scale (one capture each, after the bench warm-up)
O=gpurun_out/r01p; mkdir -p $O
timeout 3000 ncu --set full --clock-control none -k regex:gather_bulk -s 8 -c 1 -o $O/gather_c3 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_gather_c3.log 2>&1
