# attention epilogue probes: staging without the store instruction (wrong output) and evict_first L2 hint on the stores
for rep in 1 2; do
  echo "== base"; ATTN_CASES=gpt3 timeout 300 python scripts/bench_attn.py 2>&1 | tail -1; ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -1
  echo "== notma (probe)"; AB_LIB=paper_2209_02341_b200/lib/ab/notma.so ATTN_CASES=gpt3 timeout 300 python scripts/bench_attn.py 2>&1 | tail -1; AB_LIB=paper_2209_02341_b200/lib/ab/notma.so ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -1
  echo "== evict_first"; AB_LIB=paper_2209_02341_b200/lib/ab/hint.so ATTN_CASES=gpt3 timeout 300 python scripts/bench_attn.py 2>&1 | tail -1; AB_LIB=paper_2209_02341_b200/lib/ab/hint.so ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -1
done
