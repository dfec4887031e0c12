# Round 2, call k: ncu source-level profile of attention v3 vs v2 (S2048 steady state + config-3 mix)
mkdir -p gpurun_out
for impl in 5 4; do
for cs in "full S2048" "gpt3"; do
  tag=$(echo "$cs" | tr -d ' ')
  ENERGON_ATTN=$impl ATTN_CASES="$cs" timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_tc -s 3 -c 1 -o gpurun_out/attn_${impl}_${tag} -f python scripts/bench_attn.py > /dev/null 2>&1
  ncu -i gpurun_out/attn_${impl}_${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_${impl}_${tag}_src.csv 2>/dev/null
  ncu -i gpurun_out/attn_${impl}_${tag}.ncu-rep --page details --csv > gpurun_out/attn_${impl}_${tag}_details.csv 2>/dev/null
  ncu -i gpurun_out/attn_${impl}_${tag}.ncu-rep --page raw --csv > gpurun_out/attn_${impl}_${tag}_raw.csv 2>/dev/null
done
done
ls -la gpurun_out/attn_*
