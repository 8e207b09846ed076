"""Summarise ncu output for profiles/ (run here, on the CPU box, after gpurun).

    python scripts/ncu_summary.py --launches gpurun_out/launches_X.csv \
        --rep gpurun_out/full_X.ncu-rep --out profiles/rNN_X

Writes <out>_launches.json (per-kernel launch count / total / mean time from
the `--metrics gpu__time_duration.sum` pass, i.e. each kernel's share of the
step) and <out>_ncu.json (key `--set full` counters per captured launch:
duration, DRAM bytes read/write, DRAM/FP64/issue utilisation, occupancy
limits, top warp-stall reasons).
"""
import argparse
import collections
import csv
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "derived__memory_l1_wavefronts_shared_excessive"]


def short(name):
    name = name.replace("void ", "").replace("bnf::", "").replace("(anonymous namespace)::", "")
    name = name.replace("unnamed>::", "")
    return name.split("(")[0]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) / 1e3
    tot = sum(v[1] for v in agg.values())
    return {"total_us": tot, "kernels": [
        {"kernel": k, "launches": v[0], "total_us": round(v[1], 2), "mean_us": round(v[1] / v[0], 2),
         "share": round(v[1] / tot, 4)} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]}


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and
             not h.endswith("not_issued")]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = float(r[i].replace(",", ""))
                except ValueError:
                    d[k] = r[i]
                if units[i]:
                    d[k + " [unit]"] = units[i]
        tot = sum(float(r[i] or 0) for i in stall) or 1.0
        top = sorted(((float(r[i] or 0) / tot, hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                      for i in stall), reverse=True)[:6]
        d["top_stalls"] = {n: round(f, 3) for f, n in top}
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    if a.launches:
        with open(a.out + "_launches.json", "w") as f:
            json.dump(launches(a.launches), f, indent=1)
    if a.rep:
        with open(a.out + "_ncu.json", "w") as f:
            json.dump(full(a.rep), f, indent=1)


if __name__ == "__main__":
    main()
