# attention v2 probe: context-row stores dropped (lib/ab/nostore.so, wrong output) vs default -- epilogue store cost
for rep in 1 2; do
  echo "== default"; ATTN_CASES=gpt3 timeout 300 python scripts/bench_attn.py 2>&1 | tail -1; ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -1
  echo "== nostore"; AB_LIB=paper_2209_02341_b200/lib/ab/nostore.so ATTN_CASES=gpt3 timeout 300 python scripts/bench_attn.py 2>&1 | tail -1; AB_LIB=paper_2209_02341_b200/lib/ab/nostore.so ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -1
done
