# stream-K finisher preload made opportunistic: correctness, QKV trace, policy sweep on TP 1-8 shapes
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "streamk or gemm" > gpurun_out/pytest_sk_r2x.log 2>&1; rc=$?; echo "sk tests rc=$rc"; tail -2 gpurun_out/pytest_sk_r2x.log
if [ $rc -ne 0 ]; then exit 1; fi
rm -f gpurun_out/trace_*.txt
ENERGON_SK_FORCE=1 ENERGON_GEMM_TRACE=gpurun_out/trace_sk_qkv.txt timeout 120 python scripts/gemm_one.py 4096 1920 5120 1 > /dev/null
python scripts/gemm_trace_sk.py gpurun_out/trace_sk_qkv.txt | head -20
for k in 8 4 2 1; do
  H=5120; T=4096
  for shape in "$T $((3*H/k)) $H 1" "$T $H $((H/k)) 0" "$T $((4*H/k)) $H 2" "$T $H $((4*H/k)) 0"; do
    line=""
    for sk in auto off force1 force2; do
      unset ENERGON_NO_STREAMK ENERGON_SK_FORCE
      case $sk in off) export ENERGON_NO_STREAMK=1;; force1) export ENERGON_SK_FORCE=1;; force2) export ENERGON_SK_FORCE=2;; esac
      r=$(timeout 60 python scripts/gemm_one.py $shape 2>&1 | tail -1 | sed 's/.*: //')
      line="$line | $sk $r"
    done
    echo "tp$k $shape $line"
  done
done 2>&1 | tee gpurun_out/gemm_sk_policy_r2x.log
unset ENERGON_NO_STREAMK ENERGON_SK_FORCE
