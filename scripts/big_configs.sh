# Configs 4 and 5 on ONE B200 at TP=1 (whole model resident): DRCE padding sweep (config 5) and a bench line (config 4)
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
CFG=opt66b ITERS=3 timeout 1500 python scripts/padding_sweep.py > gpurun_out/sweep_opt66b.jsonl 2> gpurun_out/sweep_opt66b.err; echo "sweep rc=$?"; cat gpurun_out/sweep_opt66b.jsonl; tail -3 gpurun_out/sweep_opt66b.err
timeout 1200 python bench.py --config opt30b --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_opt30b.json 2> gpurun_out/bench_opt30b.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_opt30b.json')); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['phases']['attention'], d.get('drce_ab'), d['clocks'])"
