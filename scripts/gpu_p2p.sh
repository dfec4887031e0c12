mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_p2p.py -x -q -p no:cacheprovider -o faulthandler_timeout=300 > gpurun_out/p2p.log 2>&1; echo "p2p rc=$?"; tail -30 gpurun_out/p2p.log | grep -v "^  File.*threading"
