"""From an ncu --set full report of the GEMM launches of one layer, write profiles/gemm_traffic.json:
per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) averaged over the layer's
GEMM launches, next to the algorithmic bytes (A + W + D once) of the same launches."""
import csv, io, json, subprocess, sys

rep, cfg, tp, out = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ki, ri, wi = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot, n, per = 0.0, 0, []
for d in data:
    if "gemm_tc" not in d[ki]:
        continue
    b = float(d[ri]) * scale[units[ri]] + float(d[wi]) * scale[units[wi]]
    per.append({"kernel": d[ki].split("(")[0], "dram_bytes": b})
    tot += b
    n += 1
try:
    doc = json.load(open(out))
except Exception:
    doc = {}
doc.setdefault(cfg, {})[f"tp{tp}"] = tot / max(n, 1)
doc.setdefault("_launches", {})[f"{cfg}_tp{tp}"] = per
doc["_note"] = ("per-launch dram__bytes_read.sum + dram__bytes_write.sum averaged over one layer's four GEMM "
                "launches (ncu --set full --clock-control none); keys: config -> tp -> bytes")
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc[cfg]))
