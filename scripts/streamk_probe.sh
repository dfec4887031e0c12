mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "gemm or tiny or gpt3 or opt or gpt2s" > gpurun_out/sk_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sk_tests.log
for tp in 8 4 1; do
echo "== TP $tp new"; K_TP=$tp timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
echo "== TP $tp old"; ENERGON_NO_STREAMK=1 K_TP=$tp timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
done
H=768 T=2064 timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
ENERGON_NO_STREAMK=1 H=768 T=2064 timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{"
for v in 0 1; do
if [ $v = 1 ]; then export ENERGON_NO_STREAMK=1; fi
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-ab --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench nostreamk=$v', round(d['ms_per_step'],2), round(d['phases']['gemm']['ms_per_step'],2), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done
