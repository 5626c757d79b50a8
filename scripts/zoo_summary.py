"""Summarises gpurun_out/zoo_*.ncu-rep (ncu --set full captures from scripts/kernel_zoo.py)
into gpurun_out/<round>_zoo_summary.json: per kernel launch, time, DRAM/L2 bytes, pipe
utilisations, issue activity, occupancy, store efficiency and the top stall reasons.
usage: python scripts/zoo_summary.py r2a"""
import csv, glob, io, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
KEEP = re.compile(
    r"^(gpu__time_duration\.sum|dram__bytes_(read|write)\.sum|lts__t_bytes\.sum|"
    r"lts__t_sectors_op_(read|write)\.sum|sm__pipe_(tensor|fp64|fma|alu|fmaheavy)\w*cycles_active\.avg\.pct_of_peak_sustained_active|"
    r"sm__inst_executed_pipe_(fp64|lsu|fma|alu|xu)\w*\.avg\.pct_of_peak_sustained_active|"
    r"sm__throughput\.avg\.pct_of_peak_sustained_elapsed|gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed|"
    r"lts__throughput\.avg\.pct_of_peak_sustained_elapsed|launch__registers_per_thread|"
    r"launch__grid_size|launch__block_size|sm__warps_active\.avg\.pct_of_peak_sustained_active|"
    r"sm__issue_active\.avg\.pct_of_peak_sustained_active|smsp__inst_executed\.sum|"
    r"l1tex__t_(sectors|requests)_pipe_lsu_mem_global_op_(st|ld)\.sum|"
    r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum|launch__shared_mem_per_block_dynamic|"
    r"smsp__average_warps_issue_stalled_\w+_per_issue_active\.ratio|"
    r"smsp__pcsamp_warps_issue_stalled_\w+)$")


def summarise(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        e = {"kernel": d.get("Kernel Name", "")[:100], "id": d.get("ID")}
        stalls = {}
        for k, v in d.items():
            if not KEEP.match(k):
                continue
            u = units[h.index(k)]
            if "stalled" in k:
                try:
                    fv = float(v.replace(",", ""))
                except ValueError:
                    continue
                stalls[k] = fv
                continue
            e[k] = f"{v} {u}".strip()
        top = sorted(((k, v) for k, v in stalls.items() if "per_issue_active" in k), key=lambda kv: -kv[1])[:6]
        e["top_stalls_per_issue_active"] = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): v for k, v in top}
        out.append(e)
    return out


if __name__ == "__main__":
    rnd = sys.argv[1]
    res = {"round": rnd, "source": "scripts/kernel_zoo.py under ncu --set full --clock-control none"}
    for rep in sorted(glob.glob(os.path.join(OUT, "zoo_*.ncu-rep"))):
        kind = os.path.basename(rep)[4:-8]
        res[kind] = summarise(rep)
    with open(os.path.join(OUT, f"{rnd}_zoo_summary.json"), "w") as f:
        json.dump(res, f, indent=1)
    for k, v in res.items():
        if isinstance(v, list):
            for e in v:
                print(k, e["kernel"][:60], e.get("gpu__time_duration.sum"), e.get("dram__bytes_read.sum"), e.get("dram__bytes_write.sum"))
