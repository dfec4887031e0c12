# v3 exp2 FMA-offload A/B (ATTN3_EMU keys of 32 on the FMA pipe): parity with the default build (8), then timing
mkdir -p gpurun_out
export ENERGON_ATTN=5
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel_vs_oracle" 2>&1 | tail -1
for lib in paper_2209_02341_b200/lib/ab/emu0.so paper_2209_02341_b200/lib/libenergon.so paper_2209_02341_b200/lib/ab/emu12.so paper_2209_02341_b200/lib/ab/emu16.so; do
  echo "== $lib"; AB_LIB=$lib timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== v2"; ENERGON_ATTN=4 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
