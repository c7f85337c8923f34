"""Summarise ncu captures for profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py launches <launches.csv>            -> per-kernel share table
  python scripts/ncu_summary.py full <report.ncu-rep> [name]        -> key metrics per launch
  python scripts/ncu_summary.py memory <metrics.csv> [hbm_peak] [pcie_peak]
        -> per kernel: launches, avg us, HBM / PCIe (sysmem) / NVLink (peer) GB/s
           achieved per launch vs the peaks (the csv of an ncu --metrics run with
           gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum,
           syslts__t_sectors_aperture_sysmem_lookup_miss.sum,
           syslts__t_sectors_aperture_peer_lookup_miss.sum: sectors of 32 B read from
           host memory / peer GPUs through the system L2 slice)
Prints markdown; `full` also prints one JSON line with the DRAM traffic per launch.
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
    "syslts__t_sectors_aperture_sysmem_lookup_miss.sum",
    "syslts__t_sectors_aperture_peer_lookup_miss.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
         "nsecond": 1e-9, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:70]}` | {c} | {t*1e6:.1f} | {t/tot*100:.1f}% | {t/c*1e6:.2f} |")


def full(path, name=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"report `{path.split('/')[-1]}`\n")
    print("| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |")
    print("|---" * (len(rows) - 1) + "|")
    kn = h.index("Kernel Name")
    print("| kernel | " + " | ".join(f"`{r[kn].split('(')[0]}`" for r in rows[2:]) + " |")
    dram = []
    for k in KEYS:
        if k not in h:
            continue
        i = h.index(k)
        print(f"| {k} | " + " | ".join(f"{r[i]} {units[i]}" for r in rows[2:]) + " |")
    ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    for r in rows[2:]:
        dram.append(float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]])
    print()
    print(json.dumps({"report": path.split("/")[-1], "kernel": name,
                      "dram_bytes_per_launch": [int(x) for x in dram],
                      "dram_bytes_per_launch_mean": int(sum(dram) / len(dram))}))


def memory(path, hbm_peak=6543.4, pcie_peak=55.4):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ni, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    idi = h.index("ID")
    launches_ = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[vi] in ("n/a", ""):
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        if "t_sectors" in r[ni]:
            v = float(r[vi].replace(",", "")) * 32  # sectors -> bytes
        launches_[r[idi]][r[ni]] = v
        names[r[idi]] = r[ki].split("(")[0].replace("void ", "")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for lid, m in launches_.items():
        a = agg[names[lid]]
        a["n"] += 1
        a["t"] += m.get("gpu__time_duration.sum", 0.0)
        a["hbm"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["sys"] += m.get("syslts__t_sectors_aperture_sysmem_lookup_miss.sum", 0.0)
        a["peer"] += m.get("syslts__t_sectors_aperture_peer_lookup_miss.sum", 0.0)
    print(f"| kernel | launches | avg us | HBM GB/s (of {hbm_peak:.0f}) | PCIe sysmem GB/s "
          f"(of {pcie_peak:.1f}) | NVLink peer GB/s |")
    print("|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
        t = a["t"]
        if t <= 0:
            continue
        hb, sy, pe = a["hbm"] / t / 1e9, a["sys"] / t / 1e9, a["peer"] / t / 1e9
        print(f"| `{k[:60]}` | {int(a['n'])} | {t / a['n'] * 1e6:.1f} | {hb:.0f} "
              f"({hb / hbm_peak:.2f}) | {sy:.1f} ({sy / pcie_peak:.2f}) | {pe:.1f} |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "memory":
        memory(sys.argv[2], *[float(x) for x in sys.argv[3:5]])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
