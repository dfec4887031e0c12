mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "gemm or streamk or fused_layout or tiny_vs_oracle or gpt2s" > gpurun_out/pytest_gemmtma.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -1 gpurun_out/pytest_gemmtma.log
if [ $rc -ne 0 ]; then exit 1; fi
for rep in 1 2; do
  for shape in "4096 15360 5120 1" "4096 5120 5120 0" "4096 20480 5120 2" "4096 5120 20480 0" "4096 1920 5120 1" "4096 5120 640 0" "4096 2560 5120 2" "4096 5120 2560 0"; do
    a=$(timeout 60 python scripts/gemm_one.py $shape | sed 's/.*: //')
    b=$(AB_LIB=paper_2209_02341_b200/lib/ab/gemm_tma_lane.so timeout 60 python scripts/gemm_one.py $shape | sed 's/.*: //')
    echo "rep$rep $shape | warp-tma $a | lane-tma $b"
  done
done
for rep in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline --no-ab --no-e2e --no-tp-check --steps 20 > gpurun_out/bench_ao_$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_ao_$rep.json')); print('bench rep$rep', round(d['ms_per_step'],2), round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done
