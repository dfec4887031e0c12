# N3 LN-prologue GEMM: parity (short timeout), then A/B in the bench (configs 2 and 3)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "ln_prologue" > gpurun_out/pytest_ln_r2y.log 2>&1; rc=$?; echo "ln tests rc=$rc"; tail -15 gpurun_out/pytest_ln_r2y.log
if [ $rc -ne 0 ]; then exit 1; fi
for cfg in gpt2s gpt3_13b; do
  for lf in 0 1; do
    timeout 900 python bench.py --config $cfg --ln-fuse $lf --no-cpu-baseline --no-ab --no-e2e --steps 20 > gpurun_out/bench_${cfg}_lf$lf.json 2>gpurun_out/bench_ln.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_${cfg}_lf$lf.json')); print('$cfg ln_fuse=$lf', round(d['ms_per_step'],3), round(d['value']), d['phases']['gemm'], d['phases']['memory_bound']['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
tail -3 gpurun_out/bench_ln.err
