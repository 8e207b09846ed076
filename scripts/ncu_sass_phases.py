"""Stall samples of one kernel in an ncu report, split at the kernel's
block barriers / branches into SASS segments, plus the per-pipe counters
(diagnostics for DESIGN §6c).

    python scripts/ncu_sass_phases.py REPORT.ncu-rep KERNEL_REGEX [OUT.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "l1tex__data_pipe_lsu_wavefronts.avg",
           "l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "launch__grid_size"]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    raw = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv", "-k", "regex:" + kre]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    pipes = {m: (vals[hdr.index(m)], units[hdr.index(m)]) for m in METRICS if m in hdr}
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass",
                                            "-k", "regex:" + kre]))))
    hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][-1]
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h)]
    ix = {k: i for i, k in enumerate(h)}
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(int(r[ix[key]] or 0) for r in data)
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    agg = {k[6:]: round(sum(float(r[ix[k]] or 0) for r in data) / tot, 3) for k in reasons}
    segs, acc, start = [], 0, 0
    base = int(data[0][0], 16)
    for r in data:
        a = int(r[0], 16) - base
        s = r[1].strip()
        acc += int(r[ix[key]] or 0)
        op = s.split()[1] if s.startswith("@") else (s.split()[0] if s else "")
        if op.startswith(("BAR", "BRA", "EXIT")):
            segs.append({"from": hex(start), "to": hex(a), "share": round(acc / tot, 3), "ends_with": s[:48]})
            acc, start = 0, a
    res = {"report": rep, "kernel": kre, "samples": tot,
           "stalls": dict(sorted(agg.items(), key=lambda x: -x[1])[:10]),
           "segments": [g for g in segs if g["share"] >= 0.004], "pipes": pipes}
    txt = json.dumps(res, indent=1)
    if out:
        with open(out, "w") as f:
            f.write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
