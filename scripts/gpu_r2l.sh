mkdir -p gpurun_out
rm -f gpurun_out/attn_trace_*.txt
ENERGON_ATTN_TRACE=gpurun_out/attn_trace_s2048.txt ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -2
ENERGON_ATTN_TRACE=gpurun_out/attn_trace_gpt3.txt ATTN_CASES="gpt3" timeout 300 python scripts/bench_attn.py 2>&1 | tail -2
python scripts/attn_trace_report.py gpurun_out/attn_trace_s2048.txt | head -60
python scripts/attn_trace_report.py gpurun_out/attn_trace_gpt3.txt | head -40
