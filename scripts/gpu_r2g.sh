mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "streamk or gemm" > gpurun_out/pytest_sk_r2g.log 2>&1; rc=$?; echo "sk tests rc=$rc"; tail -3 gpurun_out/pytest_sk_r2g.log
if [ $rc -ne 0 ]; then exit 1; fi
for k in 8 4 2 1; do K_TP=$k timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{" | sed "s/^/auto tp$k /"; ENERGON_NO_STREAMK=1 K_TP=$k timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{" | sed "s/^/dp   tp$k /"; done | tee gpurun_out/gemm_sk_ab_r2g.log
timeout 900 python bench.py --local-tp 8 --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp8_r2g.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_ltp8_r2g.json')); print('ltp8 auto', d['ms_per_step'], json.dumps(d['phases']['gemm']), d['clocks'])"
ENERGON_NO_STREAMK=1 timeout 900 python bench.py --local-tp 8 --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp8_dp_r2g.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_ltp8_dp_r2g.json')); print('ltp8 dp', d['ms_per_step'], json.dumps(d['phases']['gemm']), d['clocks'])"
timeout 900 python bench.py --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_r2g.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_r2g.json')); print('tp1 auto', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
ENERGON_NO_STREAMK=1 timeout 900 python bench.py --no-cpu-baseline --no-ab --no-e2e > gpurun_out/bench_dp_r2g.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_dp_r2g.json')); print('tp1 dp', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['clocks'])"
