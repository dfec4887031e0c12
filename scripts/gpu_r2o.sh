# TP=8 QKV / MLP-up shapes: tile code x stream-K policy (A/B in one process each)
mkdir -p gpurun_out
for shape in "4096 1920 5120 1" "4096 2560 5120 2" "4096 5120 2560 0" "4096 5120 640 0"; do
  for t in 1256 1192 1128; do
    for sk in auto off force1 force2; do
      unset ENERGON_NO_STREAMK ENERGON_SK_FORCE
      case $sk in off) export ENERGON_NO_STREAMK=1;; force1) export ENERGON_SK_FORCE=1;; force2) export ENERGON_SK_FORCE=2;; esac
      echo "tile $t sk $sk: $(ENERGON_GEMM_TILE=$t timeout 60 python scripts/gemm_one.py $shape 2>&1 | tail -1)"
    done
  done
done 2>&1 | tee gpurun_out/gemm_tiles_sk_r2o.log
