mkdir -p gpurun_out
export ENERGON_ATTN=5
rm -f gpurun_out/attn_trace_*.txt
ENERGON_ATTN_TRACE=gpurun_out/attn_trace_s2048.txt ATTN_CASES="full S2048" timeout 300 python scripts/bench_attn.py 2>&1 | tail -1
python scripts/attn_trace_report.py gpurun_out/attn_trace_s2048.txt 2>/dev/null | head -24
