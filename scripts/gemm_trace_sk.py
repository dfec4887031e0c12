"""Per-cluster timelines of one traced pair-GEMM launch (ENERGON_GEMM_TRACE, last launch in the file):
units (kind W/E/F, k-blocks), MMA issue window, gaps, epilogue windows; cluster finish spread."""
import sys
from collections import defaultdict

launches = []
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        launches.append((line.strip(), []))
    elif launches and line.strip():
        f = list(map(int, line.split()))
        launches[-1][1].append(f)
hdr, recs = launches[-1]
t0min = min(r[4] for r in recs)
cl = defaultdict(list)
for c, u, tile, nkb, t0, t1, t2, e0, e1, kind in recs:
    cl[c].append((u, tile, nkb, (t0 - t0min) / 1e3, (t1 - t0min) / 1e3, (t2 - t0min) / 1e3,
                  (e0 - t0min) / 1e3 if e0 else 0, (e1 - t0min) / 1e3 if e1 else 0, "WEF"[kind]))
fin = {c: max(max(x[7], x[5]) for x in v) for c, v in cl.items()}
mma_busy = {c: sum(x[5] - x[4] for x in v) for c, v in cl.items()}
print(hdr, f"clusters {len(cl)} span {max(fin.values()):.1f} us, finish min {min(fin.values()):.1f} "
      f"median {sorted(fin.values())[len(fin) // 2]:.1f}; MMA-busy median {sorted(mma_busy.values())[len(fin) // 2]:.1f} us")
for c in sorted(cl)[:3] + sorted(cl)[len(cl) // 2:len(cl) // 2 + 1] + sorted(cl)[-3:]:
    print(f" cluster {c}: finish {fin[c]:.1f}")
    prev_t2 = None
    for u, tile, nkb, t0, t1, t2, e0, e1, k in sorted(cl[c]):
        gap = f" gap {t0 - prev_t2:5.1f}" if prev_t2 is not None else ""
        print(f"   u{u} {k} tile {tile:4d} kb {nkb:3d}: acq {t0:6.1f} first {t1:6.1f} last-issue {t2:6.1f}{gap}"
              f" | epi {e0:6.1f}-{e1:6.1f}")
        prev_t2 = t2
