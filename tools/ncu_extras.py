"""Reduce the per-op `ncu --set full --page raw --csv` exports written by
tools/profile_extras.sh to one JSON: for every op, each launch's duration,
DRAM read/write bytes, L2 hit rate, issue-active and the top stall, plus the
op's algorithmic bytes so traffic / algorithmic is explicit.

    python tools/ncu_extras.py gpurun_out/prof_r02 > profiles/r02_extras_traffic.json
"""
import csv
import json
import sys
from pathlib import Path

N, M = 232_965, 114_497_502
P, I, F = 8, 4, 4


def algorithmic(op, d):
    if op in ("copy_sum",):
        return (N + 1) * P + M * I + M * d * F + N * d * F
    if op == "copy_max":
        return (N + 1) * P + M * I + M * d * F + N * d * F + N * d * 8
    if op == "umul_sum":
        return (N + 1) * P + 2 * M * I + M * d * F + M * F + N * d * F
    if op == "dot_sddmm":
        return 2 * M * I + 2 * M * d * F + M * F
    if op == "softmax":
        return (N + 1) * P + M * I + 2 * M * d * F
    if op == "softmax_bwd":  # reads alpha and d alpha, writes ds
        return (N + 1) * P + M * I + 3 * M * d * F
    return None


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1, "ms": 1e-3,
         "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "%": 1}
STALLS = ["long_scoreboard", "lg_throttle", "wait", "short_scoreboard", "math_pipe_throttle",
          "barrier", "mio_throttle", "not_selected", "no_instruction", "membar"]


def load(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]

    def val(r, name):
        if name not in h:
            return None
        i = h.index(name)
        try:
            return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        except ValueError:
            return None

    out = []
    for r in rows[2:]:
        stall = {s: val(r, "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s)
                 for s in STALLS}
        stall = {k: v for k, v in stall.items() if v is not None}
        top = max(stall, key=stall.get) if stall else None
        out.append({
            "kernel": r[h.index("Kernel Name")][:100],
            "ms": round(val(r, "gpu__time_duration.sum") * 1e3, 4),
            "dram_read": val(r, "dram__bytes_read.sum"),
            "dram_write": val(r, "dram__bytes_write.sum"),
            "l2_hit_pct": val(r, "lts__t_sector_hit_rate.pct"),
            "dram_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": val(r, "launch__registers_per_thread"),
            "top_stall": top,
        })
    return out


def main():
    d = Path(sys.argv[1])
    res = {"graph": "reference power_law(232965, 492, 0): n=%d m=%d" % (N, M),
           "note": "ncu --set full --clock-control none, one op call per capture (replay: cold "
                   "cache, serialised); dram = dram__bytes_read.sum + dram__bytes_write.sum",
           "ops": {}}
    for f in sorted(d.glob("*_raw.csv")):
        name = f.name[:-len("_raw.csv")]
        op, _, feat = name.rpartition("_d")
        launches = load(f)
        if not launches:
            continue
        dram = sum((x["dram_read"] or 0) + (x["dram_write"] or 0) for x in launches)
        ms = sum(x["ms"] for x in launches)
        alg = algorithmic(op, int(feat))
        res["ops"][name] = {
            "launches": launches, "ms_serialised": round(ms, 4), "dram_bytes": dram,
            "algorithmic_bytes": alg,
            "dram_over_algorithmic": round(dram / alg, 3) if alg else None,
            "dram_gbs": round(dram / (ms * 1e-3) / 1e9, 1) if ms else None,
        }
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
