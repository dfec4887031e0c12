mkdir -p gpurun_out
ENERGON_ATTN=5 timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "attention_kernel_vs_oracle" > gpurun_out/pytest_v3warp.log 2>&1; rc=$?; echo "v3 tests rc=$rc"; tail -1 gpurun_out/pytest_v3warp.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2; do
  echo "== v3 warp"; ENERGON_ATTN=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== v3 lane"; ENERGON_ATTN=5 AB_LIB=paper_2209_02341_b200/lib/ab/attn_lane.so timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
  echo "== v2 warp"; timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
done
echo "== TP8 v3 warp"; ENERGON_ATTN=5 ATTN_HK=5 timeout 300 python scripts/bench_attn.py 2>&1 | tail -5
