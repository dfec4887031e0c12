mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_p2p.py -q -p no:cacheprovider -x -k "gemm or streamk or fused_layout or tiny_vs_oracle or gpt2s or local_tp or p2p" > gpurun_out/pytest_epi.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -1 gpurun_out/pytest_epi.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2; do
  for shape in "4096 5120 5120 0" "4096 20480 5120 2" "4096 5120 20480 0" "4096 5120 640 0" "4096 2560 5120 2" "4096 5120 2560 0"; do
    a=$(timeout 60 python scripts/gemm_one.py $shape | sed 's/.*: //')
    b=$(AB_LIB=paper_2209_02341_b200/lib/ab/gemm_epi_lane.so timeout 60 python scripts/gemm_one.py $shape | sed 's/.*: //')
    echo "rep$rep $shape | epi-warp $a | epi-lane(+mma lane) $b"
  done
done
