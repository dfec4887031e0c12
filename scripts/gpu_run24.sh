timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "gemm or tiny or tp or gpt2s" > gpurun_out/pytest_g.log 2>&1; tail -2 gpurun_out/pytest_g.log
TPS=1,2,4,8 timeout 500 python scripts/sweep_tiles.py 2>&1 | head -16 | python -c "
import sys,re
for l in sys.stdin:
    m=re.match(r'(tp\d \w+) .*?\'1256\': (\d+).*\'cublas\': (\d+)', l)
    if m: print(m.group(1), m.group(2), 'cublas', m.group(3))"
