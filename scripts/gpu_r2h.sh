for t in 1256 1192 1128; do
  for sk in auto off; do
    if [ $sk = off ]; then export ENERGON_NO_STREAMK=1; else unset ENERGON_NO_STREAMK; fi
    echo "tile $t sk $sk: $(ENERGON_GEMM_TILE=$t timeout 60 python scripts/gemm_one.py 4096 1920 5120 1)"
  done
done
unset ENERGON_NO_STREAMK
for t in 1256 1192; do echo "tp4 out tile $t: $(ENERGON_GEMM_TILE=$t timeout 60 python scripts/gemm_one.py 4096 5120 1280 0)"; done
for t in 1256 1192; do echo "tp8 out tile $t: $(ENERGON_GEMM_TILE=$t timeout 60 python scripts/gemm_one.py 4096 5120 640 0)"; done
for t in 1256 1192; do echo "tp1 up tile $t: $(ENERGON_GEMM_TILE=$t timeout 60 python scripts/gemm_one.py 4096 20480 5120 2)"; done
