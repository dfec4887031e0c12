import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, synth
from gpu_helpers import SHAPES, destroy, make_engine, max_abs_rel, oracle_model, run_forward
shape = SHAPES["tiny"]
B, S, seed = 4, 16, 0
lens = synth.random_lengths(B, S, seed)
tok = synth.tokens(B, S, shape["V"], lens, seed)
for dtype in ("bf16", "f32"):
  for causal in (0, 1):
    layers, emb = oracle_model(shape, seed, dtype)
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"], causal=causal)
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    errs = []
    outs = []
    for rep in range(int(os.environ.get("REPS", 3))):
        ctxs = make_engine(shape, seed, dtype, B * S, drce=1, causal=causal)
        y = run_forward(ctxs, tok, lens, dtype, shape["H"])
        destroy(ctxs)
        errs.append(max_abs_rel(y, ref, lens))
        outs.append(y)
    same = all(np.array_equal(outs[0], o) for o in outs)
    print(dtype, "causal", causal, "errs", ["%.3e" % e for e in errs], "bit-identical runs:", same, flush=True)
