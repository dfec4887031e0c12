timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout=300 -k "graph" 2>&1 | tail -3
for g in 1 0; do
timeout 300 python bench.py --config gpt2s --steps 20 --warmup 5 --no-cpu-baseline --no-ab --graph $g 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('gpt2s graph=$g', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'])"
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-ab --graph $g 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('gpt3 graph=$g', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'])"
done
