"""GPU test of the P2P TP exchange (cfg.comm = ENERGON_COMM_P2P): two or eight processes, one context each,
peers' exchange regions mapped by CUDA IPC, handles all-gathered over torch.distributed (gloo).  The
single-GPU pool runs both ranks on cuda:0 (IPC works between processes of one device; the GPU
time-slices the two contexts), which exercises the same signal / reduce / push / wait protocol an
8-GPU box runs over NVLink.  Bars: both ranks hold bit-identical outputs, they equal
the in-device local-group run of the same sequence-parallel schedule bit for bit, and they match the
fp64 oracle within the north-star tolerances."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"f32": 1e-4, "bf16": 2e-2}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, dtype, q, case="random"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import torch.distributed as dist

        import synth
        from gpu_helpers import SHAPES, load_engine, torch_dtype
        from paper_2209_02341_b200 import energon
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        energon.load_library()
        shape = _shape(case)
        B, S, seed, lens = _case(case)
        tok = torch.from_numpy(synth.tokens(B, S, shape["V"], lens, seed)).cuda()
        cfg = energon.make_config(shape["L"], shape["H"], shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S,
                                  dtype=dtype, tp_size=world, tp_rank=rank, comm=energon.COMM_P2P)
        ctx = energon.energon_init(cfg)
        load_engine([ctx], shape, seed, dtype)
        out = torch.full((B, S, shape["H"]), float("nan"), dtype=torch_dtype(dtype), device="cuda")
        res = {"rank": rank}
        try:
            energon.energon_forward(ctx, tok, lens, out)
        except energon.EnergonError as e:
            res["not_connected_status"] = e.status
        handles = [None] * world
        dist.all_gather_object(handles, energon.energon_p2p_handle(ctx))
        energon.energon_p2p_connect(ctx, handles)
        ys = []
        for _ in range(2):  # two forwards: the epochs and the self-resetting counters carry over
            out.fill_(float("nan"))
            energon.energon_forward(ctx, tok, lens, out)
            energon.energon_sync(ctx)
            ys.append(out.float().cpu().numpy())
        res["y"] = ys
        res["stats"] = energon.energon_get_stats(ctx)
        dist.barrier()
        energon.energon_destroy(ctx)
        dist.destroy_process_group()
        q.put(res)
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put({"rank": rank, "exc": repr(e), "tb": traceback.format_exc()})


def _case(case):
    """(B, S, seed, lens): random lengths, or a single 1-token sequence (T = 1 < k: rank 1's shard is
    empty, its kernels still take part in the completion protocol), or a wider model whose row-parallel
    GEMMs run on the 2-CTA tcgen05 kernel and so store their rows straight into the owners' slots (the
    fused GEMM -> reduce-scatter)."""
    import synth
    if case == "one_token":
        return 1, 4, 4, [1]
    if case in ("wide", "wide8"):
        return 8, 64, 5, synth.random_lengths(8, 64, 5)
    return 5, 33, 4, synth.random_lengths(5, 33, 4)


def _shape(case):
    from gpu_helpers import SHAPES
    if case == "wide":
        return dict(SHAPES["tiny"], L=2, H=256, h=4, F=1024, V=300, max_seq=64)
    if case == "wide8":  # 8 heads of d = 64: one head and 256 FFN columns per rank at k = 8
        return dict(SHAPES["tiny"], L=2, H=512, h=8, F=2048, V=300, max_seq=64)
    return dict(SHAPES["tiny"], L=2, V=300, max_seq=40)


@pytest.mark.parametrize("dtype,case,world", [("bf16", "random", 2), ("f32", "random", 2), ("bf16", "one_token", 2),
                                              ("bf16", "wide", 2), ("bf16", "wide8", 8), ("f32", "wide8", 8)])
def test_p2p_processes_one_gpu(dtype, case, world):
    """world = 2, and world = 8 (the north-star TP degree: 8 peers' regions mapped, 8 per-destination
    store maps in the fused GEMM -> reduce-scatter, 8-way flags) -- all processes on cuda:0."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import oracle
    import synth
    from gpu_helpers import SHAPES, destroy, make_engine, max_abs_rel, oracle_model, run_forward
    from paper_2209_02341_b200 import build, energon
    build()
    synth.build(device=True)
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_rank, args=(r, world, port, dtype, q, case)) for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=300) for _ in range(world)]
    [p.join(60) for p in procs]
    res = {r["rank"]: r for r in res}
    for r in range(world):
        assert "exc" not in res[r], res[r].get("tb")
        assert res[r]["not_connected_status"] == -7
        assert res[r]["stats"]["allreduce_calls"] == 2 * 2 * 2  # 2 per layer, 2 layers, 2 forwards
        # the wide model's row-parallel GEMMs run on the 2-CTA kernel: every exchange is GEMM -> RS fused
        assert res[r]["stats"]["fused_exchanges"] == (8 if case.startswith("wide") and dtype == "bf16" else 0)
    y0 = res[0]["y"]
    for r in range(1, world):  # bit-identical replicas
        assert np.array_equal(y0[0], res[r]["y"][0]) and np.array_equal(y0[1], res[r]["y"][1])
    assert np.array_equal(y0[0], y0[1])                                    # run to run
    # same schedule in one process (local group, in-device rank-order reduce-scatter / all-gather)
    energon.load_library()
    shape = _shape(case)
    B, S, seed, lens = _case(case)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    ctxs = make_engine(shape, seed, dtype, B * S, k=world)
    try:
        for c in ctxs:
            energon.energon_set_option(c, energon.OPT_TP_SP, 1)
        ylocal = run_forward(ctxs, tok, lens, dtype, shape["H"])
    finally:
        destroy(ctxs)
    assert np.array_equal(y0[0].astype(np.float64), ylocal)
    layers, emb = oracle_model(shape, seed, dtype)
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    ref = oracle.forward_padded(cfg, layers, emb, tok, lens)
    assert max_abs_rel(y0[0].astype(np.float64), ref, lens) <= TOL[dtype]
    for b, n in enumerate(lens):
        assert not y0[0][b, n:].any()
