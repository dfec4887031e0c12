timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "pmep or tiny" 2>&1 | tail -2
timeout 900 python scripts/pmep_bench.py > gpurun_out/pmep.log 2>&1; cat gpurun_out/pmep.log
