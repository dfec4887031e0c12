timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph" 2>&1 | tail -1
timeout 120 python scripts/bench_attn.py 2>&1 | tail -4
bash scripts/attn_trace.sh > gpurun_out/attn_trace_report.txt; tail -3 gpurun_out/attn_trace_report.txt
