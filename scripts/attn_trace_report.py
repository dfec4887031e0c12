"""Timeline of attention v3's first tiles on CTA 0 (ENERGON_ATTN_TRACE output): per slot and tile, clocks
relative to the first record -- S seen by softmax, P handed over, P seen by the MMA thread, next S issued."""
import sys
launches, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        cur = []; launches.append((line.strip(), cur))
    else:
        cur.append(list(map(int, line.split())))
name, recs = launches[-1]
t0 = min(r[2] for r in recs)
print(name)
print("slot tile   S_seen  P_done  (softmax)  MMA_Pseen (lag)  issued (issue)  | next S_seen - issued | ld max exp st")
by = {(r[0], r[1]): r for r in recs}
for (k, n), r in sorted(by.items(), key=lambda x: x[1][2]):
    nx = by.get((k, n + 1))
    print(f"{k:4d} {n:4d} {r[2]-t0:8d} {r[3]-t0:8d} ({r[3]-r[2]:6d}) {r[4]-t0:8d} ({r[4]-r[3]:5d}) {r[5]-t0:8d} ({r[5]-r[4]:5d})"
          + (f"  | {nx[2]-r[5]:6d}" if nx else "  |       ")
          + (f" | {r[6]-r[2]:5d} {r[7]-r[6]:5d} {r[8]-r[7]:5d} {r[9]-r[8]:5d}" if len(r) > 6 and r[6] else ""))
