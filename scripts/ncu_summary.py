"""Summarise ncu --set full captures into one JSON (the profiles/ evidence).

    python scripts/ncu_summary.py OUT.json name=path.ncu-rep [name=path.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]


def summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name", "")}
    for k in KEYS:
        if k in d:
            out[k] = f"{d[k]} {u.get(k, '')}".strip()
    stalls = {}
    for k in hdr:
        if "smsp__average_warps_issue_stalled" in k and k.endswith("_per_issue_active.ratio"):
            try:
                v = float(d[k] or 0)
            except ValueError:
                continue
            if v > 0.1:
                stalls[k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")] = round(v, 3)
    out["stalls_per_issue"] = stalls
    return out


def main():
    out = {"source": "ncu --set full --clock-control none --import-source on, one launch each "
                     "(scripts/gpu_r2*.sh), units as ncu reports them"}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        out[name] = summary(rep)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
