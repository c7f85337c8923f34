#!/bin/bash
O=gpurun_out/${1:-r01g2}; mkdir -p $O
timeout 1800 python bench.py --config c3 --steps 100 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 2400 python bench.py --config c4 --steps 100 --warmup 5 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
