"""DRAM traffic of the conv kernels over one c2 tick, from an ncu CSV
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
-k regex:"conv_|chain_") -> profiles/ncu_conv_summary.json (read by bench.py):
per kernel (K4c = chain_pp, K4b = conv_pp, K4 = conv_tc) and the per-layer
convs together."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, mi, ui, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
per = collections.defaultdict(dict)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
for r in data:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    per[r[ii]]["kernel"] = r[ki].split("(")[0]
def summ(name):
    launches = [v for v in per.values() if name in v["kernel"]]
    rd = sum(v.get("dram__bytes_read.sum", 0) for v in launches)
    wr = sum(v.get("dram__bytes_write.sum", 0) for v in launches)
    ns = sum(v.get("gpu__time_duration.sum", 0) for v in launches)
    return {"launches": len(launches), "dram_read_bytes_per_tick": rd, "dram_write_bytes_per_tick": wr,
            "dram_bytes_per_tick": rd + wr, "dram_bytes_per_launch": (rd + wr) / max(1, len(launches)),
            "ncu_ms_per_tick_cold": ns / 1e6}


out = {"source": sys.argv[1], "note": "ncu serialises launches with cold caches; compare shares, not absolute times",
       "chain_pp": summ("chain_pp"), "conv_pp": summ("conv_pp"), "conv_tc": summ("conv_tc"),
       "all_conv": summ("conv_")}
# the dominant kernel at top level: the K4c chain launch when the tick ran it, else K4b
out.update(out["chain_pp"] if out["chain_pp"]["launches"] else out["conv_pp"])
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
