# Round 2, call b: device-side lengths / work list + bucketed graphs; GEMM TP shapes vs cuBLAS; local TP=8 step.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_r2b.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_r2b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r2b.json 2>gpurun_out/bench_r2b.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_r2b.json')); print('gpt3 seeds', d['value'], d['ms_per_step'], d['per_seed'], d['e2e']['value'], d['roofline']['achieved'])"
for cfg in gpt2s; do
 for sd in 5 1; do
  timeout 600 python bench.py --config $cfg --seeds $sd --no-cpu-baseline --no-ab --steps 20 > gpurun_out/bench_${cfg}_s${sd}.json 2>>gpurun_out/bench_r2b.err; python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_s${sd}.json')); print('$cfg seeds=$sd', d['value'], d['ms_per_step'], d['per_seed']['ms_median'], d['e2e']['ms_per_step'])"
 done
done
for k in 1 2 4 8; do K_TP=$k timeout 300 python scripts/bench_gemm.py 2>&1 | grep -v "^{" ; done | tee gpurun_out/gemm_vs_cublas_r2b.log
timeout 900 python bench.py --local-tp 8 --no-cpu-baseline --no-ab --no-e2e --steps 5 > gpurun_out/bench_ltp8_r2b.json 2>>gpurun_out/bench_r2b.err; python -c "
import json; d=json.load(open('gpurun_out/bench_ltp8_r2b.json')); print('ltp8', d['ms_per_step'], json.dumps(d['phases']), d['clocks'])"
