mkdir -p gpurun_out
python scripts/gemm_one.py 4096 5120 1280 0
ENERGON_NO_STREAMK=1 python scripts/gemm_one.py 4096 5120 1280 0
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -s 5 -c 1 -o gpurun_out/sk_tp4out -f python scripts/gemm_one.py 4096 5120 1280 0 > /dev/null 2>&1
ncu -i gpurun_out/sk_tp4out.ncu-rep --page source --csv --print-source sass > gpurun_out/sk_src.csv 2>/dev/null
ncu -i gpurun_out/sk_tp4out.ncu-rep --page details --csv > gpurun_out/sk_details.csv 2>/dev/null
ls -la gpurun_out/sk_*
