"""profiles/ncu_traffic.json from an `ncu --set full --page raw --csv` export of
one bench step (tools/profile_round.sh): DRAM bytes of every launch of the
step, summed (the step is pack + one row-kernel launch per column tile +
unpack), plus the L2 hit rate and L2 sector traffic of the row kernel.

python tools/ncu_traffic.py gpurun_out/prof/step_raw.csv ROUND FEAT EDGES NODES"""
import csv
import json
import sys

raw, rnd, feat, edges, nodes = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), \
    int(sys.argv[5])
rows = list(csv.reader(open(raw)))
h, units = rows[0], rows[1]


def col(name):
    return h.index(name)


def val(r, name):
    i = col(name)
    v = float(r[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1, "ms": 1e-3,
             "us": 1e-6, "ns": 1e-9, "%": 1}.get(u, 1)
    return v * scale


launches = []
for r in rows[2:]:
    launches.append({
        "kernel": r[col("Kernel Name")][:80],
        "ms": val(r, "gpu__time_duration.sum") * 1e3,
        "dram_read": val(r, "dram__bytes_read.sum"),
        "dram_write": val(r, "dram__bytes_write.sum"),
        "l2_hit_pct": val(r, "lts__t_sector_hit_rate.pct"),
        "l2_read_sectors": val(r, "lts__t_sectors_srcunit_tex_op_read.sum"),
    })
step = [x for x in launches if "spmm_rows" in x["kernel"] or "pack_tiles" in x["kernel"]]
row = [x for x in step if "spmm_rows" in x["kernel"]]
alg = (nodes + 1) * 8 + edges * 4 + edges * feat * 4 + nodes * feat * 4
out = {
    "round": rnd,
    "kernel": "spmm_rows_kernel<float,COPY,SUM,V=4,MP_F> x %d column tiles + pack/unpack" % len(row),
    "workload": "reddit_spmm_copy_u_sum", "feat": feat, "edges": edges, "nodes": nodes,
    "launches_per_step": len(step),
    "dram_bytes_read": sum(x["dram_read"] for x in step),
    "dram_bytes_write": sum(x["dram_write"] for x in step),
    "dram_bytes_per_launch": sum(x["dram_read"] + x["dram_write"] for x in step),
    "algorithmic_bytes_per_launch": alg,
    "row_kernel_l2_hit_pct": sum(x["l2_hit_pct"] for x in row) / max(1, len(row)),
    "row_kernel_l2_read_bytes": sum(x["l2_read_sectors"] for x in row) * 32,
    "row_kernel_dram_bytes_per_launch": sum(x["dram_read"] + x["dram_write"] for x in row)
    / max(1, len(row)),
    "row_kernel_l2_read_bytes_per_launch": sum(x["l2_read_sectors"] for x in row) * 32
    / max(1, len(row)),
    "serialized_ms": sum(x["ms"] for x in step),
    "per_launch": step,
    "note": "per_launch is one bench step (ncu replay, cold cache); dram_bytes_per_launch is the "
            "whole step: the step is the unit bench.py times",
}
json.dump(out, sys.stdout, indent=1)
print()
