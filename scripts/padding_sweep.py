"""Padding-ratio sweep of the DRCE A/B on one B200 (BASELINE config 5's sweep p in {0,.25,.5,.75}):
DRCE on vs off latency and valid tok/s.  CFG=gpt3_13b (default) or opt30b / opt66b (the whole model at
TP=1 fits the 180 GB of one B200: 130 GB of bf16 weights for OPT-66B); ITERS timed forwards per point."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2209_02341_b200 import energon

cfgname = os.environ.get("CFG", "gpt3_13b")
shape = dict(synth.SHAPES[cfgname])
if os.environ.get("LAYERS"):
    shape["L"] = int(os.environ["LAYERS"])
B, S = synth.BATCHES[cfgname]["B"], synth.BATCHES[cfgname]["S"]
H = shape["H"]
energon.load_library()
cfg = energon.make_config(shape["L"], H, shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S)
ctx = energon.energon_init(cfg)
emb = {n: synth.emb_tensor_device(n, H, shape["V"], shape["max_seq"], 0, True, torch.bfloat16) for n in synth.EMB_TENSORS}
energon.energon_load_embeddings(ctx, emb["tok_emb"], emb["pos_emb"], emb["lnf_g"], emb["lnf_b"])
for l in range(shape["L"]):
    w = {n: synth.layer_tensor_device(n, l, H, shape["F"], 0, True, torch.bfloat16) for n in synth.LAYER_TENSORS}
    energon.energon_load_layer_weights(ctx, l, w)
    del w
out = torch.empty(B, S, H, dtype=torch.bfloat16, device="cuda")
rows = []
for p in (0.0, 0.25, 0.5, 0.75):
    lens = synth.exact_p_lengths(B, S, p, 0)
    T = sum(lens)
    tok = torch.from_numpy(synth.tokens(B, S, shape["V"], lens, 0)).cuda()
    res = {"config": cfgname, "layers": shape["L"], "p": p, "T": T}
    for drce in (1, 0):
        energon.energon_set_option(ctx, energon.OPT_DRCE, drce)
        for _ in range(2):
            energon.energon_forward(ctx, tok, lens, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        iters = int(os.environ.get("ITERS", "5"))
        for _ in range(iters):
            energon.energon_forward(ctx, tok, lens, out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res["on_ms" if drce else "off_ms"] = ms
        res["on_tok_s" if drce else "off_tok_s"] = T / ms * 1e3
    res["latency_reduction"] = 1 - res["on_ms"] / res["off_ms"]
    rows.append(res)
    print(json.dumps(res), flush=True)
energon.energon_destroy(ctx)
