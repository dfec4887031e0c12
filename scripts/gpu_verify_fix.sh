mkdir -p gpurun_out
for i in 1 2; do
timeout 250 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "streamk or graph or pmep or tiny" > gpurun_out/fix_subset_$i.log 2>&1; echo "subset $i rc=$?"; tail -1 gpurun_out/fix_subset_$i.log
done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_fix.json 2>gpurun_out/bench_fix.err; python -c "
import json; d=json.load(open('gpurun_out/bench_fix.json')); print(d['value'], d['ms_per_step'], d['phases']['attention'], d['roofline']['achieved'], d['clocks'])"
