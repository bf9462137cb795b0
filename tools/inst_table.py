"""Warp instructions per bench step of the ALU-bound secondary configs, from the ncu launch lists
written by tools/gpu/ncu_inst.sh (bench.py --config X --steps 1 --warmup 3 under ncu), into
profiles/ncu_instructions.json, which bench.py reads for the issue roofline of those lines.

A step is one call of the timed function; under ncu it runs warmup + steps times (+1 for the
result read-back call GREEDY and MERIT make after timing).  Kernels of other libraries (torch
input generation) are excluded by name; GREEDY's two workloads are told apart by grid size.
   python tools/inst_table.py gpurun_out"""
import collections
import csv
import json
import re
import sys

CASES = {  # name: (csv, kernel regex, grids or None, executions of the timed function)
    "C2": ("inst_C2.csv", r"fused_sweep_kernel|finalize_kernel", None, 4),
    "MERIT": ("inst_MERIT.csv", r"merit_kernel", None, 5),
    "SSIM": ("inst_SSIM.csv", r"ssim_fused_kernel", None, 4),
    "GREEDY D2": ("inst_GREEDY.csv", r"digits_kernel|score_kernel|search_kernel", {"(1526, 1, 1)", "(720, 1, 1)"}, 5),
    "GREEDY D1": ("inst_GREEDY.csv", r"digits_kernel|score_kernel|search_kernel", {"(26, 1, 1)", "(40320, 1, 1)"}, 5),
}


def main(d):
    out = {"unit": "warp-instructions per step (smsp__inst_executed.sum)",
           "source": "tools/gpu/ncu_inst.sh + tools/inst_table.py"}
    for name, (fn, pat, grids, execs) in CASES.items():
        rows = [r for r in csv.DictReader(l for l in open(f"{d}/{fn}") if not l.startswith("=="))]
        tot = 0.0
        per = collections.Counter()
        for r in rows:
            if r.get("Metric Name") != "smsp__inst_executed.sum" or not re.search(pat, r["Kernel Name"]):
                continue
            if grids is not None and r["Grid Size"] not in grids:
                continue
            v = float(r["Metric Value"].replace(",", ""))
            tot += v
            per[re.search(pat, r["Kernel Name"]).group(0)] += 1
        out[name] = {"warp_inst_per_step": tot / execs, "launches": dict(per), "executions": execs}
    json.dump(out, open("profiles/ncu_instructions.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
