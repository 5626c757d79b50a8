"""Builds profiles/<round>_ncu_summary.json from a round's captures:
gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch list) and
gpurun_out/prof.ncu-rep (ncu --set full of the hot kernels).
usage: python scripts/ncu_summary.py r1b "<bench command>" """
import csv, io, json, os, subprocess, sys
from collections import defaultdict
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__issue_active.avg.pct_of_peak_sustained_active"]

def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    acc = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            acc[r[ki][:80]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in acc.values())
    return {k: {"launches": len(v), "avg_us": sum(v) / len(v) / 1e3 if max(v) > 1e3 else sum(v) / len(v),
                "share": sum(v) / tot} for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1]))}

def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        e = {"kernel": d.get("Kernel Name", "")[:80]}
        for m in METRICS:
            if m in d:
                e[m] = d[m]
        out.append(e)
    return out

if __name__ == "__main__":
    rnd, cmd = sys.argv[1], sys.argv[2]
    res = {"round": rnd, "command": cmd}
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        res["launch_list_avg"] = launch_list(os.path.join(OUT, "launches.csv"))
    if os.path.exists(os.path.join(OUT, "prof.ncu-rep")):
        res["ncu_full"] = full(os.path.join(OUT, "prof.ncu-rep"))
    if os.path.exists(os.path.join(OUT, "prof_action.ncu-rep")):
        res["ncu_full_action"] = full(os.path.join(OUT, "prof_action.ncu-rep"))
    dest = os.environ.get("NCU_SUMMARY_DIR", os.path.join(ROOT, "profiles"))
    with open(os.path.join(dest, f"{rnd}_ncu_summary.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])
