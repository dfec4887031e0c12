timeout 400 python -m pytest tests/test_gpu_pipeline.py -x -q -p no:cacheprovider -o faulthandler_timeout=300 > gpurun_out/pp_dist.log 2>&1; echo "rc=$?"; tail -25 gpurun_out/pp_dist.log
