# ncu --set full with source of the tcgen05 attention (config-3 length mix) for stall analysis
mkdir -p gpurun_out
cat > /tmp/attn_one.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2209_02341_b200 import energon
energon.load_library()
B, S, hk, d = 16, 512, 40, 128
lens = synth.exact_p_lengths(B, S, 0.5, 0)
Q, K, V = (torch.randn(B, hk, S, d, device="cuda").bfloat16() for _ in range(3))
O = torch.empty_like(Q)
for _ in range(4):
    energon.energon_attention(Q, K, V, O, lens, 1)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_tc2 -s 2 -c 1 -o gpurun_out/attn_prof -f python /tmp/attn_one.py > /dev/null 2>&1
ncu -i gpurun_out/attn_prof.ncu-rep --page source --csv --print-source sass > gpurun_out/attn_src.csv 2>/dev/null
ncu -i gpurun_out/attn_prof.ncu-rep --page details --csv > gpurun_out/attn_details.csv 2>/dev/null
ls -la gpurun_out/attn_*
