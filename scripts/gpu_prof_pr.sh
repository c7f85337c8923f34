# ncu of one full K3 step on C2: launch list + full captures of both kernels
O=gpurun_out/${1:-prof_pr}; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/pr_launches.csv python scripts/pr_probe.py c2 full > $O/pr_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pr_step -s 1 -c 1 -o $O/light python scripts/pr_probe.py c2 full > $O/ncu_light.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pr_hub -s 1 -c 1 -o $O/hub python scripts/pr_probe.py c2 full > $O/ncu_hub.log 2>&1
