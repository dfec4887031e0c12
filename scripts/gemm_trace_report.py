"""Summarise ENERGON_GEMM_TRACE output (last launch of each shape): per unit-round durations of the
pair GEMM's MMA issuer, first-data latency, and the spread of cluster finish times."""
import sys
from collections import defaultdict

launches = []
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        launches.append((line.strip(), []))
        splits = []
    elif line.startswith("split"):
        _, c, a, b, cc, d, flag = line.split()
        a, b, cc, d, flag = int(a), int(b), int(cc), int(d), int(flag)
        print(f"  split piece (cluster {c}): fence+barrier+atomic {(b - a) / 1e3:.2f} us, "
              f"{'reduce+store' if flag >> 32 else 'wait'} {(cc - b) / 1e3:.2f} us, final barrier {(d - cc) / 1e3:.2f} us,"
              f" nsplit {flag & 0xffffffff}") if (flag >> 32) else None
    elif launches:
        c, u, tile, nkb, t0, t1, t2, e0, e1 = map(int, line.split())
        launches[-1][1].append((c, u, tile, nkb, t0, t1, t2, e0, e1))
last = {}
for hdr, recs in launches:
    last[hdr] = recs
for hdr, recs in last.items():
    tmin = min(r[4] for r in recs)
    by_u = defaultdict(list)
    fin = defaultdict(int)
    for c, u, tile, nkb, t0, t1, t2, e0, e1 in recs:
        by_u[u].append((t0 - tmin, t1 - t0, t2 - t0, (e1 - e0) if e1 else 0, nkb))
        fin[c] = max(fin[c], (e1 if e1 else t2) - tmin)
    print(hdr, f"span {max(fin.values()) / 1e3:.1f} us")
    for u in sorted(by_u):
        v = by_u[u]
        print(f"  round {u}: units {len(v):3d}  start {min(x[0] for x in v) / 1e3:6.1f}-{max(x[0] for x in v) / 1e3:6.1f} us"
              f"  first-data wait {sum(x[1] for x in v) / len(v) / 1e3:5.2f} us  issue span {sum(x[2] for x in v) / len(v) / 1e3:6.2f} us"
              f"  epilogue {sum(x[3] for x in v) / len(v) / 1e3:6.2f} (max {max(x[3] for x in v) / 1e3:6.2f}) us  kb {min(x[4] for x in v)}-{max(x[4] for x in v)}")
    f = sorted(fin.values())
    print(f"  cluster finish: min {f[0] / 1e3:.1f}  median {f[len(f) // 2] / 1e3:.1f}  max {f[-1] / 1e3:.1f} us")
