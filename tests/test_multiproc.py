"""World-size-2 gloo tests of the N>1 host path on the CPU: unique-id / seq_lens broadcast, the
library's shard plan driving a real two-process TP layer (oracle partials + gloo allreduce), the
2-reductions-per-layer count, and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2209_02341_b200 import dist as edist
        from paper_2209_02341_b200 import energon
        out = {}
        # (1) NCCL-unique-id style broadcast and the engine command's lengths
        uid = edist.broadcast_bytes(bytes(range(128)) if rank == 0 else None, 128)
        lens = edist.broadcast_lengths([5, 3, 7] if rank == 0 else [1], 0)
        out["uid_ok"] = uid == bytes(range(128))
        out["lens"] = lens
        # (2) one TP layer across the 2 processes, sliced by the library's own shard plan
        L, H, h, F = 1, 32, 4, 128
        cfg = energon.make_config(L, H, h, F, 64, 16, 64, dtype="f32", tp_size=world, tp_rank=rank)
        plan = energon.energon_shard_plan(cfg)
        layers, emb = synth.model_host(L, H, F, 64, 16, 5, False)
        w = layers[0]
        B, S = len(lens), max(lens)
        tok = synth.tokens(B, S, 64, lens, 5)
        ocfg = oracle.make_cfg(L, H, h, F)
        X = oracle.embed(ocfg, emb, tok)
        reductions = 0
        # attention module: this rank's heads (columns of wq/wk/wv, rows of wo) per the plan
        c0, nc = plan["qkv_col0"], plan["qkv_cols"]
        shard = dict(w)
        for n in ("wq", "wk", "wv"):
            shard[n] = np.ascontiguousarray(w[n][:, c0:c0 + nc])
        for n in ("bq", "bk", "bv"):
            shard[n] = np.ascontiguousarray(w[n][c0:c0 + nc])
        shard["wo"] = np.ascontiguousarray(w["wo"][c0:c0 + nc, :])
        f0, nf = plan["ffn_col0"], plan["ffn_cols"]
        shard["w1"] = np.ascontiguousarray(w["w1"][:, f0:f0 + nf])
        shard["b1"] = np.ascontiguousarray(w["b1"][f0:f0 + nf])
        shard["w2"] = np.ascontiguousarray(w["w2"][f0:f0 + nf, :])
        # the shard, run as a k=1 rank-local computation: partial = attention of own heads . wo rows
        A = oracle.layernorm(X, w["ln1_g"], w["ln1_b"])
        local = oracle.make_cfg(1, nc, plan["heads"], nf)
        Q = A.reshape(-1, H) @ shard["wq"] + shard["bq"]
        K = A.reshape(-1, H) @ shard["wk"] + shard["bk"]
        V = A.reshape(-1, H) @ shard["wv"] + shard["bv"]
        C = oracle.attention(Q.reshape(B, S, nc), K.reshape(B, S, nc), V.reshape(B, S, nc), plan["heads"], lens)
        part = torch.from_numpy(oracle.matmul(C.reshape(-1, nc), shard["wo"]))
        dist.all_reduce(part)  # "accumulated by communications"
        reductions += 1
        X1 = X + part.numpy().reshape(B, S, H) + w["bo"]
        A2 = oracle.layernorm(X1, w["ln2_g"], w["ln2_b"])
        G = oracle.matmul(A2.reshape(-1, H), shard["w1"]) + shard["b1"]
        G = np.vectorize(oracle.gelu)(G)
        part2 = torch.from_numpy(oracle.matmul(G, shard["w2"]))
        dist.all_reduce(part2)
        reductions += 1
        X2 = X1 + part2.numpy().reshape(B, S, H) + w["b2"]
        ref = oracle.layer_padded(ocfg, w, X, lens)
        out["err"] = max(float(np.abs(X2[b, :n] - ref[b, :n]).max()) for b, n in enumerate(lens))
        out["reductions"] = reductions
        out["plan"] = plan
        # (3) max over ranks
        out["max"] = edist.max_over_ranks(float(rank + 1))
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def test_two_process_tp_layer_gloo():
    from paper_2209_02341_b200 import build
    build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in res[r], res[r].get("error")
        assert res[r]["uid_ok"]
        assert res[r]["lens"] == [5, 3, 7]
        assert res[r]["reductions"] == 2  # one synchronisation per pair of linears
        assert res[r]["err"] < 1e-12, res[r]["err"]
        assert res[r]["max"] == 2.0
    assert res[0]["plan"]["head0"] == 0 and res[1]["plan"]["head0"] == 2
    assert res[0]["plan"]["ffn_col0"] == 0 and res[1]["plan"]["ffn_col0"] == 64
