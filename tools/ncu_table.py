"""Build profiles/ncu_inst.json (read by bench.py for the issue view of the roofline) and a
per-round summary from tools/ncu_table.sh's exported raw pages.

    python tools/ncu_table.py <tag>        # reads gpurun_out/ncu_<tag>/*.raw.csv

Per workload: the dominant roll-out kernel's warp instructions per launch
(smsp__inst_executed.sum), issue-active % (per active SMSP, and per SM over the elapsed time),
warps active, DRAM bytes, pipe utilisation (fma / fp64 / alu / xu), stall ratios and the
store coalescing ratio."""
import csv
import glob
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import wsinputs as W  # noqa: E402

tag = sys.argv[1]
src = f"gpurun_out/ncu_{tag}"
KEEP = {
    "gpu__time_duration.sum": "duration_us",
    "smsp__inst_executed.sum": "inst_per_launch",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "sm_issue_elapsed_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "pipe_fp64_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "launch__registers_per_thread": "registers",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "lanes_per_inst",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum": "st_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum": "st_requests",
}
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3}
table, summary = {}, {}
for f in sorted(glob.glob(os.path.join(src, "*.raw.csv"))):
    name = os.path.basename(f)[:-8]
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")], "grid": v[h.index("Grid Size")], "block": v[h.index("Block Size")]}
    stalls = {}
    for i, n in enumerate(h):
        if n in KEEP:
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            d[KEEP[n]] = x * SCALE.get(u[i], 1.0) if n.startswith("dram__bytes") or n.startswith("gpu__time") else x
        elif n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                stalls[n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
            except ValueError:
                pass
    d["stalls_per_issue"] = {k: round(x, 3) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]) if x >= 0.01}
    if d.get("st_requests"):
        d["st_sectors_per_request"] = round(d["st_sectors"] / d["st_requests"], 2)
    d["dram_bytes"] = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
    w = W.CONFIGS.get(name)
    E = w.n_envs if w else None
    summary[name] = d
    table[name] = {"E": E, "kernel": d["kernel"], "inst_per_launch": d.get("inst_per_launch"),
                   "issue_active_pct": d.get("issue_active_pct"), "sm_issue_elapsed_pct": d.get("sm_issue_elapsed_pct"),
                   "dram_bytes": d["dram_bytes"],
                   "source": f"ncu --set full, profiles/{tag}/ncu_summary.json"}
os.makedirs(f"profiles/{tag}", exist_ok=True)
json.dump(summary, open(f"profiles/{tag}/ncu_summary.json", "w"), indent=1)
path = "profiles/ncu_inst.json"
old = json.load(open(path)) if os.path.exists(path) else {}
old.update(table)
json.dump(old, open(path, "w"), indent=1, sort_keys=True)
for k, d in summary.items():
    print(f"{k:5s} {d['duration_us']:9.1f} us  inst {d.get('inst_per_launch', 0):.3g}  issue(active) "
          f"{d.get('issue_active_pct', 0):5.1f}%  sm-issue(elapsed) {d.get('sm_issue_elapsed_pct', 0):5.1f}%  "
          f"warps {d.get('warps_active_pct', 0):5.1f}%  fma {d.get('pipe_fma_pct', 0):4.1f} fp64 "
          f"{d.get('pipe_fp64_pct', 0):4.1f} alu {d.get('pipe_alu_pct', 0):4.1f} xu {d.get('pipe_xu_pct', 0):4.1f}  "
          f"dram {d['dram_bytes'] / 1e6:.0f} MB  regs {d.get('registers')}")
