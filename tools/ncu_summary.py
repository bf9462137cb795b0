"""Summaries of ncu output for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches gpurun_out/launches.csv      # per-kernel share of the step
    python tools/ncu_summary.py full gpurun_out/x.ncu-rep [algorithmic_bytes_per_launch]
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second", "launch__shared_mem_per_block_dynamic",
]


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("adct::<unnamed>::", "").replace("void ", "")
    return name[:90]


def launches(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"]) + f"  grid={r['Grid Size']}"
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        v = v * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print(f"{'kernel':95s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:95s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:9.1f} {100 * v / s:5.1f}%")
    print(f"{'TOTAL':95s} {sum(cnt.values()):8d} {s:10.1f}")


def full(path, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = csv.reader(io.StringIO(out))
    hdr = next(rd)
    units = next(rd)
    for row in rd:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print("kernel:", short(d.get("Kernel Name", "?")), " grid", d.get("Grid Size"), " block", d.get("Block Size"))
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        print("  warp-state samples (share):", ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:8]))
        if alg_bytes:
            try:
                rb = float(d["dram__bytes_read.sum"].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u["dram__bytes_read.sum"]]
                wb = float(d["dram__bytes_write.sum"].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u["dram__bytes_write.sum"]]
                print(f"  traffic = {rb + wb:.6g} B per launch; algorithmic = {alg_bytes:.6g} B; ratio {(rb + wb) / alg_bytes:.4f}")
            except Exception as e:  # noqa: BLE001
                print("  traffic: n/a", e)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None)
