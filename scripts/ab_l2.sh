# A/B of GEMM L2 policies in the full bench step (GPT-3-13B TP=1): A-panel group budget and D-store hints
mkdir -p gpurun_out
run() { env $1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-ab --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), round(d['phases']['gemm']['ms_per_step'],2), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
run ENERGON_GROUP_MB=48
run ENERGON_GROUP_MB=96
run ENERGON_GROUP_MB=200
run ENERGON_L2_HINTS=2
run "ENERGON_L2_HINTS=2 ENERGON_GROUP_MB=96"
done
export ENERGON_PROFILE_RANGE=1
for v in "ENERGON_GROUP_MB=48" "ENERGON_GROUP_MB=96" "ENERGON_L2_HINTS=2 ENERGON_GROUP_MB=96"; do
env $v timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:gemm -c 8 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ab --layers 2 --graph 0 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; 
ki,mn,mv=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
for r in rows[1:]:
    print('$v', r[ki][:28], r[mn], r[mv])" | tail -12
done
