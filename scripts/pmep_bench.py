"""PMEP (peer memory pooling, PAPER.md:375-424 / sec 5.6) on one B200 with a pinned-host pool: step
time of the GPT-3-13B-shape stack (40 layers, B=16, S=512, p=0.5) with `resident` layers on the GPU and
the rest placed by energon_pmep_plan and prefetched over PCIe on a copy stream."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2209_02341_b200 import energon

energon.load_library()
name = os.environ.get("CFG", "gpt3_13b")
shape = dict(synth.SHAPES[name])
B, S = synth.BATCHES[name]["B"], synth.BATCHES[name]["S"]
H, L = shape["H"], shape["L"]
lens = synth.batch_lengths(name, 0)
T = sum(lens)
tok = torch.from_numpy(synth.tokens(B, S, shape["V"], lens, 0)).cuda()
out = torch.empty(B, S, H, dtype=torch.bfloat16, device="cuda")

# raw pinned-host -> device bandwidth for reference
hb = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
db = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
db.copy_(hb, non_blocking=True); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    db.copy_(hb, non_blocking=True)
torch.cuda.synchronize()
h2d = 3 * (1 << 30) / (time.perf_counter() - t0) / 1e9
del hb, db
print(json.dumps({"h2d_GBps": h2d}), flush=True)


def build():
    cfg = energon.make_config(L, H, shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S)
    ctx = energon.energon_init(cfg)
    emb = {n: synth.emb_tensor_device(n, H, shape["V"], shape["max_seq"], 0, True, torch.bfloat16) for n in synth.EMB_TENSORS}
    energon.energon_load_embeddings(ctx, emb["tok_emb"], emb["pos_emb"], emb["lnf_g"], emb["lnf_b"])
    for l in range(L):
        w = {n: synth.layer_tensor_device(n, l, H, shape["F"], 0, True, torch.bfloat16) for n in synth.LAYER_TENSORS}
        energon.energon_load_layer_weights(ctx, l, w)
        del w
    return ctx


def time_steps(ctx, n=5):
    for _ in range(2):
        energon.energon_forward(ctx, tok, lens, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        energon.energon_forward(ctx, tok, lens, out)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


ctx = build()
base = time_steps(ctx)
energon.energon_destroy(ctx)
layer_bytes = 12 * H * H * 2
print(json.dumps({"resident": L, "ms": base, "valid_tok_s": T / base * 1e3}), flush=True)
for resident, slots in ((36, 1), (36, 2), (32, 2), (30, 3)):
    ctx = build()
    plan = energon.energon_pmep_plan(L, resident)
    energon.energon_offload_layers(ctx, plan, slots=slots, pool=0)
    ms = time_steps(ctx)
    st = energon.energon_get_stats(ctx)
    energon.energon_destroy(ctx)
    per_layer_compute = base / L
    xfer = layer_bytes / (h2d * 1e9) * 1e3
    print(json.dumps({"resident": resident, "offloaded": plan, "slots": slots, "ms": ms,
                      "throughput_loss": 1 - base / ms, "per_layer_compute_ms": per_layer_compute,
                      "per_layer_transfer_ms_pcie": xfer,
                      "per_layer_transfer_ms_nvlink_770GBps": layer_bytes / 770e9 * 1e3,
                      "prefetch_GB": st["prefetch_bytes"] / 1e9}), flush=True)
