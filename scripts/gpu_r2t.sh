# (1) sanitizers on the attention kernels incl. v3 (ENERGON_ATTN=5) and the round-2 GEMM stream-K;
# (2) in-step A/B: stream-K tail vs data parallel at TP=1 (power-capped step), alternating
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for impl in 4 5; do
    ENERGON_ATTN=$impl timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -m gpu \
      -k "attention_kernel_vs_oracle or tiny_vs_oracle or streamk" -p no:cacheprovider > gpurun_out/sanitize_${tool}_attn$impl.log 2>&1
    echo "$tool attn=$impl exit $?"; tail -2 gpurun_out/sanitize_${tool}_attn$impl.log
  done
done
for rep in 1 2; do
  for sk in on off; do
    if [ $sk = off ]; then export ENERGON_NO_STREAMK=1; else unset ENERGON_NO_STREAMK; fi
    timeout 900 python bench.py --no-cpu-baseline --no-ab --no-e2e --no-tp-check --steps 20 > gpurun_out/bench_sk_${sk}_$rep.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/bench_sk_${sk}_$rep.json')); print('sk=$sk rep=$rep', round(d['ms_per_step'],2), round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
  done
done
unset ENERGON_NO_STREAMK
