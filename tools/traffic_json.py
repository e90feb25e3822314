"""Summarise an ncu capture of the bench into profiles/traffic_cfg3.json:
per kernel, DRAM bytes read+written and duration of one launch."""
import csv, json, subprocess, sys
rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic_cfg3.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
res = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    key = next((v for k, v in (("k_backward_points", "points_bwd"), ("k_gather", "gather"),
                               ("k_scatter_emit", "scatter_emit"), ("k_count_red", "count"), ("k_count_smem", "count"),
                               ("k_bbox_validate", "bbox")) if k in name), name[:40])
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
             "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}

    def g(m):
        if m not in h:
            return None
        k = h.index(m)
        return float(r[k].replace(",", "")) * scale.get(units[k], 1.0)
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    res[key] = {"kernel": name[:80], "dram_read_bytes": rd, "dram_write_bytes": wr,
                "traffic_bytes": rd + wr if rd is not None else None,
                "duration_us_ncu": g("gpu__time_duration.sum")}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
