# attention v2: L2 prefetch of only the next item's Q / K_0 / V_0 (default here) vs none (lib/ab/nopf.so)
for rep in 1 2; do
  echo "== prefetch (softmax warp)"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== none"; AB_LIB=paper_2209_02341_b200/lib/ab/nopf.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
