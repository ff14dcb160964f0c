"""Summarise ncu captures (gpurun_out/*.ncu-rep) and the launch list into profiles/<tag>/.

    python tools/profile_summary.py <tag>

Writes <kernel>_metrics.json (selected raw metrics), <kernel>_stalls.json (stall mix and
instruction mix from the source page), launches_summary.json (per-kernel share of the step
from the gpu__time_duration launch list), and updates profiles/traffic.json (dram bytes per
launch of the roll-out kernel, read by bench.py as roofline.traffic)."""
import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "latest"
out = os.path.join("profiles", tag)
os.makedirs(out, exist_ok=True)
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "sm__cycles_elapsed.avg", "lts__t_bytes.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    return raw_rows(list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv")))))


def raw_rows(rows):
    if len(rows) < 3:
        return {}
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else ""}
        for n in WANT:
            if n in h:
                i = h.index(n)
                d[n] = {"value": v[i], "unit": u[i]}
        res.append(d)
    return res


def source_mix(rep):
    return source_rows(list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")))))


def source_rows(rows):
    if len(rows) < 3:
        return {}
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) >= len(h) - 1]
    stalls, ops = collections.Counter(), collections.Counter()
    for d in data:
        for c in h:
            if c.startswith("stall_") and "Not Issued" not in c:
                try:
                    stalls[c] += int(d[c] or 0)
                except ValueError:
                    pass
        s = d.get("Source", "").strip().split()
        if s:
            op = s[1] if s[0].startswith("@") else s[0]
            ops[op.split(".")[0]] += int(d.get("Instructions Executed") or 0)
    ts = sum(stalls.values()) or 1
    to = sum(ops.values()) or 1
    return {"stall_pct": {k: round(100 * v / ts, 1) for k, v in stalls.most_common()},
            "warp_instructions": to,
            "op_mix_pct": {k: round(100 * v / to, 1) for k, v in ops.most_common(25)}}


def to_bytes(m, key):
    return float(m[key]["value"]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m[key]["unit"]]


summary = {}
captures = [(os.path.basename(r)[len("prof_"):-len(".ncu-rep")], r, None) for r in sorted(glob.glob("gpurun_out/prof_*.ncu-rep"))]
# captures exported to csv on the GPU box (tools/prof_one.sh, tools/prof_envs.sh)
captures += [(os.path.basename(r)[len("prof_"):-len(".raw.csv")], None, r) for r in sorted(glob.glob("gpurun_out/prof_*.raw.csv"))]
for name, rep, rawcsv in captures:
    if rep:
        m = raw_metrics(rep)
        s = source_mix(rep)
    else:
        m = raw_rows(list(csv.reader(open(rawcsv))))
        src = rawcsv[:-len(".raw.csv")] + ".src.csv"
        s = source_rows(list(csv.reader(open(src)))) if os.path.exists(src) else {}
        if name.startswith("env_") and m:  # per-workload roll-out capture: record its traffic
            tf = "profiles/traffic.json"
            t = json.load(open(tf)) if os.path.exists(tf) else {}
            wl = name[len("env_"):]
            t[wl] = to_bytes(m[0], "dram__bytes_read.sum") + to_bytes(m[0], "dram__bytes_write.sum")
            t[wl + "_source"] = f"profiles/{tag}/{name}_metrics.json (ncu --set full, one launch)"
            json.dump(t, open(tf, "w"), indent=1)
    json.dump(m, open(os.path.join(out, f"{name}_metrics.json"), "w"), indent=1)
    json.dump(s, open(os.path.join(out, f"{name}_stalls.json"), "w"), indent=1)
    summary[name] = {"metrics": m, "stalls": s}
    if name == "rollout" and m:
        rd = float(m[0]["dram__bytes_read.sum"]["value"]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m[0]["dram__bytes_read.sum"]["unit"]]
        wr = float(m[0]["dram__bytes_write.sum"]["value"]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m[0]["dram__bytes_write.sum"]["unit"]]
        tf = "profiles/traffic.json"
        t = json.load(open(tf)) if os.path.exists(tf) else {}
        t["C2"] = rd + wr
        t["C2_source"] = f"profiles/{tag}/rollout_metrics.json (ncu --set full, one launch of k_rollout_discrete, C2)"
        json.dump(t, open(tf, "w"), indent=1)

if os.path.exists("gpurun_out/launches.csv"):
    rows = list(csv.reader(open("gpurun_out/launches.csv")))
    st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[st]
    d = collections.defaultdict(list)
    for r in rows[st + 1:]:
        if len(r) >= len(h):
            x = dict(zip(h, r))
            d[x["Kernel Name"]].append(float(x["Metric Value"]))
    tot = sum(sum(v) for v in d.values())
    ls = {k: {"launches": len(v), "mean_us": round(sum(v) / len(v) / 1e3, 2), "share": round(sum(v) / tot, 4)}
          for k, v in d.items()}
    json.dump(ls, open(os.path.join(out, "launches_summary.json"), "w"), indent=1)
    summary["launches"] = ls
    import shutil
    shutil.copy("gpurun_out/launches.csv", os.path.join(out, "launches.csv"))
for f in ("bench.json", "sweep.jsonl", "pytest_gpu.log"):
    if os.path.exists(f"gpurun_out/{f}"):
        import shutil
        shutil.copy(f"gpurun_out/{f}", os.path.join(out, f))
print(json.dumps({k: (v if k == "launches" else v["stalls"].get("stall_pct", {})) for k, v in summary.items()}, indent=1)[:3000])
