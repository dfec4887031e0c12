"""GPU tests of the pipeline stage entry (energon_forward_stage, NBPP PAPER.md:302-346) and of the
in-process pipeline on one B200: stage contexts that hold only their own layers, chained with PACKED
activations, against the fp64 oracle (north-star tolerances) and against each other (the pipelined
run must equal the sequential chain of the same stages bit for bit)."""
import random
import threading

import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import SHAPES, destroy, load_engine, max_abs_rel, oracle_model, torch_dtype

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_02341_b200 import build, energon
    build()
    energon.load_library()
    synth.build(device=True)


def E():
    from paper_2209_02341_b200 import energon
    return energon


def make_stages(shape, seed, dtype, max_tokens, pp, k=1, drce=1):
    """One context (or local TP group of k) per stage, each loaded with its own layer range only."""
    e = E()
    ranges = e.energon_stage_plan(shape["L"], pp)
    stages = []
    for a, b in ranges:
        cfg = e.make_config(shape["L"], shape["H"], shape["h"], shape["F"], shape["V"], shape["max_seq"], max_tokens,
                            dtype=dtype, drce=drce)
        ctxs = [e.energon_init(cfg)] if k == 1 else e.energon_init_local_group(cfg, k)
        load_engine(ctxs, shape, seed, dtype, layers=range(a, b))
        stages.append((ctxs, a, b))
    return stages


def run_chain(stages, tok_np, lens, dtype, H, drce=1):
    """The stages one after the other on the current stream (no pipelining)."""
    e = E()
    B, S = tok_np.shape
    tok = torch.from_numpy(tok_np).cuda()
    rows = sum(lens) if drce else B * S
    x = None
    for i, (ctxs, a, b) in enumerate(stages):
        last = i == len(stages) - 1
        if last:
            out = torch.full((B, S, H), float("nan"), dtype=torch_dtype(dtype), device="cuda")
        else:
            out = torch.full((rows, H), float("nan"), dtype=torch.float32, device="cuda")
        kind = e.STAGE_FINAL if last else e.STAGE_PACKED
        kw = dict(tokens=tok if i == 0 else None, x=x)
        if len(ctxs) == 1:
            e.energon_forward_stage(ctxs[0], lens, S, a, b, kind, out, **kw)
        else:
            e.energon_forward_stage_group(ctxs, lens, S, a, b, kind, out, **kw)
        x = out
    torch.cuda.synchronize()
    return x


def reference(shape, seed, dtype, tok, lens):
    layers, emb = oracle_model(shape, seed, dtype)
    cfg = oracle.make_cfg(shape["L"], shape["H"], shape["h"], shape["F"])
    return oracle.forward_padded(cfg, layers, emb, tok, lens)


def as_np(y):
    return y.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("pp,k", [(2, 1), (3, 1), (2, 2)])
@pytest.mark.parametrize("drce", [1, 0])
def test_stage_chain_vs_oracle(dtype, pp, k, drce):
    shape = dict(SHAPES["tiny"], L=3, V=300, max_seq=40)
    B, S, seed = 5, 33, 6
    lens = synth.random_lengths(B, S, seed)
    tok = synth.tokens(B, S, shape["V"], lens, seed)
    stages = make_stages(shape, seed, dtype, B * S, pp, k=k, drce=drce)
    try:
        y = as_np(run_chain(stages, tok, lens, dtype, shape["H"], drce=drce))
        for ctxs, _, _ in stages:  # a stage context holds only its own layers
            with pytest.raises(E().EnergonError) as ei:
                out = torch.empty((B, S, shape["H"]), dtype=torch_dtype(dtype), device="cuda")
                E().energon_forward(ctxs[0], torch.from_numpy(tok).cuda(), lens, out) if k == 1 else \
                    E().energon_forward_group(ctxs, torch.from_numpy(tok).cuda(), lens, out)
            assert ei.value.status == -7
    finally:
        for ctxs, _, _ in stages:
            destroy(ctxs)
    ref = reference(shape, seed, dtype, tok, lens)
    assert max_abs_rel(y, ref, lens) <= TOL[dtype]
    for b, n in enumerate(lens):
        assert not y[b, n:].any()


def test_stage_entry_validation():
    shape = dict(SHAPES["tiny"], L=2)
    e = E()
    cfg = e.make_config(2, shape["H"], shape["h"], shape["F"], shape["V"], shape["max_seq"], 64, dtype="f32")
    ctx = e.energon_init(cfg)
    try:
        w = {n: synth.layer_tensor_device(n, 1, shape["H"], shape["F"], 0, False, torch.float32)
             for n in synth.LAYER_TENSORS}
        e.energon_load_layer_weights(ctx, 1, w)  # layer 1 only, no embeddings
        lens = [3, 2]
        x = torch.zeros((5, shape["H"]), device="cuda")
        out = torch.zeros((5, shape["H"]), device="cuda")
        tok = torch.ones((2, 4), dtype=torch.int32, device="cuda")
        cases = [
            (dict(tokens=tok, x=x), 1, 2, e.STAGE_PACKED, -1),   # both inputs
            (dict(), 1, 2, e.STAGE_PACKED, -1),                  # neither
            (dict(x=x), 1, 1, e.STAGE_PACKED, -1),               # empty middle stage
            (dict(x=x), 0, 2, e.STAGE_PACKED, -7),               # layer 0 not loaded
            (dict(tokens=tok), 1, 2, e.STAGE_PACKED, -7),        # first stage needs the embeddings
            (dict(x=x), 1, 2, e.STAGE_FINAL, -7),                # last stage needs the final LN
            (dict(x=x), 1, 2, 7, -1),                            # bad out_kind
        ]
        for kw, a, b, kind, status in cases:
            with pytest.raises(e.EnergonError) as ei:
                e.energon_forward_stage(ctx, lens, 4, a, b, kind, out, **kw)
            assert ei.value.status == status, (kw.keys(), a, b, kind)
        e.energon_forward_stage(ctx, lens, 4, 1, 2, e.STAGE_PACKED, out, x=x)  # the valid middle stage runs
        e.energon_sync(ctx)
        assert torch.isfinite(out).all()
    finally:
        e.energon_destroy(ctx)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("pp", [2, 4])
def test_local_pipeline_gpu(dtype, pp):
    """NBPP on one GPU: pp stage threads, each on its own CUDA stream, 16 random batches (B in [1,8],
    S in {8,16,33}) submitted by 4 concurrent callers with injected admission delays -> every result
    equals the sequential chain of the same stages bit for bit and the oracle within tolerance; every
    stage ran the keys in order; pp - 1 transfers per batch."""
    from paper_2209_02341_b200 import pipeline as pl
    shape = dict(SHAPES["tiny"], L=4, V=300, max_seq=40)
    seed, H = 9, shape["H"]
    stages = make_stages(shape, seed, dtype, 8 * 40, pp)
    rng = random.Random(pp)
    batches = []
    for i in range(16):
        B, S = rng.randint(1, 8), rng.choice([8, 16, 33])
        lens = [rng.randint(1, S) for _ in range(B)]
        batches.append((synth.tokens(B, S, shape["V"], lens, 40 + i), lens))
    try:
        seq = [as_np(run_chain(stages, tok, lens, dtype, H)) for tok, lens in batches]
        trace = pl.Trace()
        runners = [pl.EnergonStageRunner(ctxs, a, b, first=i == 0, last=i == pp - 1, hidden=H,
                                         out_dtype=torch_dtype(dtype)) for i, (ctxs, a, b) in enumerate(stages)]
        p = pl.LocalPipeline(runners, admit_delay=0.002, lane_delay=0.002, seed=pp, trace=trace)
        futs = [None] * len(batches)

        def submitter(j):
            for i in range(j, len(batches), 4):
                futs[i] = p.submit(*batches[i])

        ts = [threading.Thread(target=submitter, args=(j,)) for j in range(4)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        outs = [as_np(f.result(timeout=120)) for f in futs]
        p.shutdown(timeout=60)
    finally:
        for ctxs, _, _ in stages:
            destroy(ctxs)
    for s in range(pp):
        assert trace.keys(s) == list(range(len(batches)))
    assert p.transfers == (pp - 1) * len(batches)
    for (tok, lens), y, ys in zip(batches, outs, seq):
        assert np.array_equal(y, ys)
        ref = reference(shape, seed, dtype, tok, lens)
        assert max_abs_rel(y, ref, lens) <= TOL[dtype]


def _dist_stage(rank, world, port, dtype, q):
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import random as rnd

        import torch.distributed as dist

        import synth
        from gpu_helpers import SHAPES, load_engine, torch_dtype
        from paper_2209_02341_b200 import energon
        from paper_2209_02341_b200 import pipeline as pl
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cmd_group, res_group = dist.new_group(backend="gloo"), dist.new_group(backend="gloo")
        energon.load_library()
        shape = dict(SHAPES["tiny"], L=4, V=300, max_seq=40)
        H, seed = shape["H"], 9
        a, b = energon.energon_stage_plan(shape["L"], world)[rank]
        cfg = energon.make_config(shape["L"], H, shape["h"], shape["F"], shape["V"], shape["max_seq"], 8 * 40,
                                  dtype=dtype)
        ctx = energon.energon_init(cfg)
        load_engine([ctx], shape, seed, dtype, layers=range(a, b))
        link = pl.DistLink(world, 1, act_spec=lambda c: ((c.rows(), H), torch.float32, "cuda:0"),
                           out_spec=lambda c: ((c.batch, c.max_len, H), torch_dtype(dtype), "cuda:0"),
                           cmd_group=cmd_group, act_group=None, res_group=res_group, stage_via_host=True)
        trace = pl.Trace()
        runner = pl.EnergonStageRunner(ctx, a, b, first=rank == 0, last=rank == world - 1, hidden=H,
                                       out_dtype=torch_dtype(dtype))
        worker = pl.StageWorker(rank, world, runner, link, admit_delay=0.002, trace=trace, seed=rank).start()
        res = {"rank": rank}
        if rank == 0:
            engine = pl.Engine(link, 2 * world, lane_delay=0.002, seed=3)
            link.engine = engine
            link.start_results()
            r = rnd.Random(5)
            batches = []
            for i in range(10):
                B, S = r.randint(1, 8), r.choice([8, 16, 33])
                lens = [r.randint(1, S) for _ in range(B)]
                batches.append((synth.tokens(B, S, shape["V"], lens, 70 + i), lens))
            futs = [engine.submit(*bt) for bt in batches]
            res["outs"] = [f.result(timeout=120).float().cpu().numpy() for f in futs]
            res["batches"] = batches
            engine.shutdown()
            link.join_results(30)
        worker.join(60)
        res.update(keys=trace.keys(rank), transfers=worker.transfers,
                   error=repr(worker.error) if worker.error else None)
        dist.barrier()
        energon.energon_destroy(ctx)
        dist.destroy_process_group()
        q.put(res)
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put({"rank": rank, "exc": repr(e), "tb": traceback.format_exc()})


@pytest.mark.parametrize("dtype", ["bf16"])
def test_dist_pipeline_two_processes_one_gpu(dtype):
    """NBPP across processes with GPU stages: stage 0 and stage 1 in two processes (both on cuda:0),
    commands from the engine on rank 0 over gloo, packed activations between the processes (through
    host memory, since both share the GPU), results back to rank 0; every result equals the
    sequential chain of the same stages bit for bit, keys in order on both stages, 1 transfer per
    batch."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_dist_stage, args=(r, world, port, dtype, q)) for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=300) for _ in range(world)]
    [p.join(60) for p in procs]
    res = {r["rank"]: r for r in res}
    for r in range(world):
        assert "exc" not in res[r], res[r].get("tb")
        assert res[r]["error"] is None
        assert res[r]["keys"] == list(range(10))
    assert res[0]["transfers"] == 10 and res[1]["transfers"] == 0
    shape = dict(SHAPES["tiny"], L=4, V=300, max_seq=40)
    stages = make_stages(shape, 9, dtype, 8 * 40, world)
    try:
        for (tok, lens), y in zip(res[0]["batches"], res[0]["outs"]):
            ys = as_np(run_chain(stages, tok, lens, dtype, shape["H"]))
            assert np.array_equal(y.astype(np.float64), ys)
    finally:
        for ctxs, _, _ in stages:
            destroy(ctxs)
