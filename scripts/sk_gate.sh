for g in 160 64; do
  for shape in "4096 5120 5120 0" "4096 5120 2560 0" "4096 10240 5120 2" "4096 5120 10240 0" "4096 2560 5120 2"; do
    ENERGON_SK_MIN_NKB=$g python scripts/gemm_one.py $shape | sed "s/^/gate=$g /"
  done
done
