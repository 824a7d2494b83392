"""ncu DRAM-traffic CSV (--metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum -k regex:k_ix_product, one launch per product at the
bench configuration) -> the JSON bench.py reads as roofline.traffic.

    python tools/traffic_json.py gpurun_out/r02_traffic_config4.csv profiles/r02_traffic_config4.json "<command>"
"""
import csv
import json
import sys

src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.reader(open(src)) if r]
hdr = next(r for r in rows if r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
alg = 65536 * 262144 * 4
out = {"command": cmd, "config": "config 4 (m=65536, n=262144, r=64), one launch of each product (k_ix_product)",
       "algorithmic_bytes_per_launch": alg, "kernels": {}}
for d in data:
    name = "A = M W^T" if "<0>" in d["Kernel Name"] or "(bool)0" in d["Kernel Name"] else "C = V^T M"
    k = out["kernels"].setdefault(name, {})
    v = float(d["Metric Value"].replace(",", ""))
    k[{"dram__bytes_read.sum": "dram_read_bytes", "dram__bytes_write.sum": "dram_write_bytes",
       "gpu__time_duration.sum": "ncu_duration_ns"}[d["Metric Name"]]] = v
for k in out["kernels"].values():
    k["traffic_bytes"] = k["dram_read_bytes"] + k["dram_write_bytes"]
    k["traffic_over_algorithmic"] = k["traffic_bytes"] / alg
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
