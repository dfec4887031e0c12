# repeat the GPU suite to look for flaky (race) failures after the attention synchronisation change
for rep in 1 2; do
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
done
for rep in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "attention or fused or layout or tiny" 2>&1 | tail -1
done
