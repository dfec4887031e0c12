"""Summarise ncu output for profiles/: (1) a launch list CSV (gpu__time_duration per launch) into
per-kernel shares of the step, (2) an ncu --set full report into the key per-kernel metrics."""
import collections, csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[mv].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {n} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
    out.append(f"| **total** | {sum(n for n, _ in agg.values())} | {tot / 1e3:.1f} | 100% |")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    cols = [hdr.index("Kernel Name"), hdr.index("Grid Size")] + [hdr.index(k) for k in KEYS if k in hdr]
    out = ["| " + " | ".join(hdr[c] + (f" ({units[c]})" if units[c] else "") for c in cols) + " |",
           "|" + "---|" * len(cols)]
    for d in data:
        vals = [d[c] for c in cols]
        vals[0] = vals[0].split("(")[0].replace("void ", "")
        out.append("| " + " | ".join(vals) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
