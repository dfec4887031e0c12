# Serpentine K order x A-panel group budget on the MLP-down shape: time (CUDA events) and DRAM bytes (ncu).
set -u
for g in 96 130 170 200; do
  echo "group $g MB: $(ENERGON_GROUP_MB=$g timeout 120 python scripts/gemm_one.py 4096 5120 20480 0)"
  ENERGON_GROUP_MB=$g timeout 300 ncu --metrics dram__bytes_read.sum -k regex:gemm_tc2 -c 3 python scripts/gemm_one.py 4096 5120 20480 0 2>&1 | grep -E "dram__" | tail -1 | sed "s/^/group $g /"
done
