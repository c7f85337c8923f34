#!/bin/bash
# One parameterised GPU-box runner (replaces round 1's one-off gpu_*.sh).
#   bash scripts/gpu.sh <tag> <stage> [<stage> ...]
# Stages (outputs under gpurun_out/<tag>/):
#   sys            box facts: CPU, RAM, IOMMU, hugepages, /dev/shm, PCIe, clocks
#   tests          pytest -m gpu (all GPU parity tests)          smoke   __graft_entry__.smoke()
#   dist           pytest tests/test_distributed.py -m gpu
#   bench:<cfg>[:<steps>]   python bench.py --config <cfg> (ours)  -> bench_<cfg>.json
#   ref:<cfg>[:<steps>]     python bench.py --impl reference       -> ref_<cfg>.json
#   probe[:<gb>]   scripts/micro/cold_probe (cold-tier translation / CE probe)
#   hpprobe[:<gb>] scripts/micro/host_pages_probe (cold tier on 4 KB / THP / 2 MB / 1 GB host pages)
#   testk:<expr>   pytest -m gpu -k <expr>
#   launches:<cfg> ncu launch list (gpu__time_duration) of a short bench run
#   ncu_k8:<cfg>   ncu (application replay) of K8 on the cached C3/C4 inputs
#   ncu_k3:<cfg>   ncu --set full of K3 (pr_step) at <cfg>
#   ncu_k3all:<cfg> ncu --set full of every K3 kernel of one step (class A hub x2, B, C stream) at <cfg>
#   prlaunch:<cfg> per-launch time / DRAM / L2 of every K3 kernel (pr_*) at <cfg>
#   k3probe:<cfg>  scripts/k3_probe.py <cfg> over the settings in $K3_SETTINGS (';'-separated)
#   pytestf:<file> pytest -m gpu of one test file
#   sanitize       compute-sanitizer memcheck/racecheck/synccheck on small cases
#   k1probe:<cfg>  scripts/k1_probe.py: K1 atomic vs binned at <cfg>
#   k1launch:<cfg> the same under an ncu launch list (per-kernel time and DRAM bytes)
#   selprobe       selection (K4-K6) at C2/C3 sizes: ours, ncu per-kernel list, and cub's LSD sort as a yardstick
#   shared2        2-process runs on one GPU (IPC gather, PageRank exchange)
T=${1:?tag}; shift
O=gpurun_out/$T; mkdir -p $O
export PYTHONUNBUFFERED=1
run() { echo "== $* ($(date +%T))" >> $O/stages.log; }
for st in "$@"; do
  IFS=: read -r name a b <<< "$st"
  run "$st"
  case $name in
    sys)
      { lscpu; free -g; df -h /dev/shm /tmp; cat /proc/cmdline; ls /sys/class/iommu 2>&1;
        dmesg 2>/dev/null | grep -i -E "iommu|dmar|vfio" | head -40;
        cat /sys/kernel/mm/transparent_hugepage/enabled; grep -i huge /proc/meminfo;
        nvidia-smi -q | grep -i -E -A3 "PCIe Generation|Link Width|Address Translation|ATS|Addressing Mode";
        nvidia-smi -q -d CLOCK,POWER; nvidia-smi topo -m; } > $O/sys.txt 2>&1 ;;
    tests) timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log ;;
    dist) timeout 900 python -m pytest tests/test_distributed.py -x -q -m gpu > $O/pytest_dist.log 2>&1; echo "rc=$?" >> $O/pytest_dist.log ;;
    bench) timeout 2400 python bench.py --config $a --steps ${b:-100} --warmup 5 > $O/bench_$a.json 2> $O/bench_$a.err ;;
    ref) timeout 1800 python bench.py --impl reference --config $a --steps ${b:-20} --warmup 5 > $O/ref_$a.json 2> $O/ref_$a.err ;;
    probe)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cold_probe scripts/micro/cold_probe.cu &&
      timeout 900 /tmp/cold_probe ${a:-45} 3400 > $O/cold_probe.log 2>&1; echo "rc=$?" >> $O/cold_probe.log ;;
    hpprobe)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/host_pages_probe scripts/micro/host_pages_probe.cu &&
      timeout 900 /tmp/host_pages_probe ${a:-45} > $O/host_pages_probe.log 2>&1; echo "rc=$?" >> $O/host_pages_probe.log ;;
    testk) timeout 2400 python -m pytest tests -x -q -m gpu -k "$a" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log ;;
    launches) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $O/launches_$a.csv python bench.py --config $a --steps 10 --warmup 3 --no-cpu-baseline \
        > $O/launches_$a.log 2>&1 ;;
    ncu_k8)
      timeout 1200 python scripts/profile_target.py prep --config $a > $O/prof_prep_$a.log 2>&1
      timeout 3000 ncu --replay-mode application --clock-control none --import-source on \
        --section SpeedOfLight --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables \
        --section WarpStateStats --section SourceCounters --section LaunchStats --section Occupancy \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_aperture_sysmem.sum,lts__t_sectors_aperture_device.sum,lts__t_sectors_srcunit_tex_aperture_sysmem.sum \
        -k regex:gather -s 2 -c 1 -o $O/k8_$a python scripts/profile_target.py k8 --config $a --launches 3 \
        > $O/ncu_k8_$a.log 2>&1 ;;
    prlaunch) timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct \
        --clock-control none --csv -k regex:"pr_|gather_floor" --log-file $O/prlaunch_$a.csv \
        python scripts/profile_target.py k3 --config $a --launches 1 > $O/prlaunch_$a.log 2>&1 ;;
    ncu_k3all) timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"pr_(hub|step|cstream)" -s 4 -c 4 \
        -o $O/k3all_$a python scripts/profile_target.py k3 --config $a --launches 1 > $O/ncu_k3all_$a.log 2>&1 ;;
    ncu_k3) timeout 2400 ncu --set full --clock-control none --import-source on -k regex:pr_step -s 2 -c 1 \
        -o $O/k3_$a python scripts/profile_target.py k3 --config $a --launches 1 > $O/ncu_k3_$a.log 2>&1 ;;
    sanitize) bash scripts/sanitize.sh $O ;;
    k3probe) timeout 1500 python scripts/k3_probe.py $a > $O/k3probe_$a.log 2>&1 ;;
    pytestf) timeout 2400 python -m pytest tests/$a -x -q -m gpu > $O/pytest_$a.log 2>&1; echo "rc=$?" >> $O/pytest_$a.log ;;
    k1probe) timeout 1200 python scripts/k1_probe.py $a >> $O/k1probe_$a.log 2>&1 ;;
    k1launch) timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv -k regex:"k1_|indeg|exclusive|tile_|sums_" --log-file $O/k1_launches_$a.csv \
        python scripts/k1_probe.py $a > $O/k1launch_$a.log 2>&1 ;;
    selprobe)
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sort_probe scripts/micro/sort_probe.cu
      for nn in 2450000 111000000; do
        timeout 300 /tmp/sort_probe $nn >> $O/selprobe.log 2>&1
        timeout 300 python scripts/select_probe.py $nn >> $O/selprobe.log 2>&1
        timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
          --log-file $O/sel_launches_$nn.csv python scripts/select_probe.py $nn 1 >> $O/selprobe_ncu.log 2>&1
      done ;;
    shared2)
      TG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config ${a:-c1} --steps 20 --warmup 3 \
        > $O/bench_${a:-c1}_2ranks_shared.json 2> $O/bench_${a:-c1}_2ranks_shared.err ;;
    *) echo "unknown stage $st" >> $O/stages.log ;;
  esac
  echo "   done $st ($(date +%T))" >> $O/stages.log
done
ls -la $O
