ENERGON_DEBUG_SYNC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention or tiny or gpt2s" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "attention or opt or fused or gpt3 or edge or tiny or gpt2s or graph or full" 2>&1 | tail -1
timeout 120 python scripts/bench_attn.py 2>&1 | tail -4
