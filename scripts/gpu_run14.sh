timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "attention_kernel" --timeout=60 > gpurun_out/pytest_attn.log 2>&1
echo "attn exit $?"; tail -15 gpurun_out/pytest_attn.log
