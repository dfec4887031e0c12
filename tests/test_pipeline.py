"""NBPP control plane on the CPU (sec 4.2): the loop counter and consistency queue,
the in-process pipeline with stage runners built from the fp64 oracle, and the multi-process pipeline
over torch.distributed (gloo).  The oracle stages move PACKED activation rows between stages, the way
the GPU stages do; every result must equal the oracle's one-shot forward of its own batch bit for bit
(row-wise fp64 arithmetic is identical however the layers are grouped)."""
import os
import random
import socket
import threading
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2209_02341_b200 import pipeline as pl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPE = dict(L=4, H=64, h=4, F=256, V=256, max_seq=16)


# ----------------------------------------------------------------------------- counter and queue
def test_loop_counter_is_unidirectional_and_unique_under_contention():
    c = pl.LoopCounter()
    got = []
    lock = threading.Lock()

    def take():
        for _ in range(100):
            v = c.next()
            with lock:
                got.append(v)

    ts = [threading.Thread(target=take) for _ in range(16)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert sorted(got) == list(range(1600)) and c.peek() == 1600


def test_queue_reorders():
    """insert 1 then 0; two pops -> 0 then 1."""
    q = pl.ConsistencyQueue()
    q.insert(1, "b")
    q.insert(0, "a")
    assert q.pop_next(1) == (0, "a") and q.pop_next(1) == (1, "b")


def test_queue_blocks_until_the_next_key_arrives():
    """only key 2 present, local counter at 0 -> pop blocks until 0 and 1 arrive."""
    q = pl.ConsistencyQueue()
    q.insert(2, "c")
    with pytest.raises(TimeoutError):
        q.pop_next(timeout=0.05)
    threading.Timer(0.05, q.insert, (1, "b")).start()
    threading.Timer(0.10, q.insert, (0, "a")).start()
    assert [q.pop_next(2)[0] for _ in range(3)] == [0, 1, 2]


@pytest.mark.parametrize("seed", range(5))
def test_queue_permutation_sweep(seed):
    """100 keys inserted in random order by concurrent threads -> pops 0..99."""
    keys = list(range(100))
    random.Random(seed).shuffle(keys)
    q = pl.ConsistencyQueue()
    chunks = [keys[i::4] for i in range(4)]
    ts = [threading.Thread(target=lambda ks=ks: [q.insert(k, k * 10) for k in ks]) for ks in chunks]
    [t.start() for t in ts]
    out = [q.pop_next(5) for _ in range(100)]
    [t.join() for t in ts]
    assert out == [(k, 10 * k) for k in range(100)]


def test_queue_rejects_duplicates_and_closes():
    q = pl.ConsistencyQueue()
    q.insert(0, "a")
    with pytest.raises(pl.ProtocolError):
        q.insert(0, "again")
    assert q.pop_next(1)[0] == 0
    with pytest.raises(pl.ProtocolError):
        q.insert(0, "stale")
    q.insert(1, "b")
    q.close()
    assert q.pop_next(1)[0] == 1  # pending keys drain after close
    with pytest.raises(pl.Closed):
        q.pop_next(1)


def test_command_rows():
    c = pl.Command(0, 0, [3, 1, 4], 5)
    assert c.batch == 3 and c.rows(True) == 8 and c.rows(False) == 15


# ----------------------------------------------------------------------------- oracle stage runners (tests only)
class OracleStage:
    """Stage [l0, l1) of the fp64 oracle with the GPU stages' interface: first stage embeds the tokens,
    the activations between stages are the packed [T, H] rows (float64 torch tensors), the last stage
    returns the final LN with pad rows 0 (DRCE output semantics)."""

    def __init__(self, model, l0, l1, first, last, delay=0.0):
        self.cfg, self.layers, self.emb = model
        self.l0, self.l1, self.first, self.last, self.delay = l0, l1, first, last, delay
        self.calls = 0

    def __call__(self, cmd, x):
        self.calls += 1
        lens, S = cmd.seq_lens, cmd.max_len
        B = len(lens)
        H = self.cfg.H
        if self.first:
            X = oracle.embed(self.cfg, self.emb, np.asarray(cmd.tokens))
        else:
            X = np.zeros((B, S, H))
            rows = x.numpy()
            assert rows.shape == (sum(lens), H)
            t = 0
            for b, n in enumerate(lens):  # rebuild padding for the oracle's padded layer stack
                X[b, :n] = rows[t:t + n]
                t += n
        X = oracle.layers_padded(self.cfg, self.layers, self.l0, self.l1, X, lens)
        if self.delay:
            time.sleep(self.delay)
        if self.last:
            Y = oracle.layernorm(X, self.emb["lnf_g"], self.emb["lnf_b"])
            for b, n in enumerate(lens):
                Y[b, n:] = 0.0
            return torch.from_numpy(Y)
        return torch.from_numpy(np.concatenate([X[b, :n] for b, n in enumerate(lens)], axis=0))


def make_model(seed=3, L=SHAPE["L"]):
    layers, emb = synth.model_host(L, SHAPE["H"], SHAPE["F"], SHAPE["V"], SHAPE["max_seq"], seed, False)
    cfg = oracle.make_cfg(L, SHAPE["H"], SHAPE["h"], SHAPE["F"])
    return cfg, layers, emb


def random_batch(rng, seed):
    B = rng.randint(1, 8)
    S = rng.choice([4, 8, 16])
    lens = [rng.randint(1, S) for _ in range(B)]
    return synth.tokens(B, S, SHAPE["V"], lens, seed), lens


def reference(model, tok, lens):
    cfg, layers, emb = model
    return oracle.forward_padded(cfg, layers, emb, tok, lens)


def assert_valid_equal(y, ref, lens):
    y = np.asarray(y)
    for b, n in enumerate(lens):
        assert np.array_equal(y[b, :n], ref[b, :n])
        assert not np.any(y[b, n:])


def plan(L, pp):
    base, rem = divmod(L, pp)
    out, b = [], 0
    for i in range(pp):
        e = b + base + (1 if i < rem else 0)
        out.append((b, e))
        b = e
    return out


# ----------------------------------------------------------------------------- in-process pipeline
def test_local_pipeline_single_batch_pp2_one_transfer():
    """pp = 2, one batch -> exactly 1 inter-stage transfer, result = the oracle."""
    model = make_model()
    runners = [OracleStage(model, a, b, i == 0, i == 1) for i, (a, b) in enumerate(plan(SHAPE["L"], 2))]
    p = pl.LocalPipeline(runners)
    tok, lens = synth.tokens(3, 8, SHAPE["V"], [8, 3, 5], 1), [8, 3, 5]
    y = p.submit(tok, lens).result(timeout=30)
    p.shutdown()
    assert p.transfers == 1
    assert_valid_equal(y, reference(model, tok, lens), lens)


def test_local_pipeline_pp1_is_serial():
    """pp = 1 -> equals serial_forward bit-exactly (degenerate pipeline)."""
    model = make_model()
    p = pl.LocalPipeline([OracleStage(model, 0, SHAPE["L"], True, True)])
    tok, lens = synth.tokens(2, 16, SHAPE["V"], [16, 9], 2), [16, 9]
    f = p.submit(tok, lens)
    y1, y2 = f.result(30), f.result(30)  # waiting twice yields the same value
    p.shutdown()
    assert y1 is y2 and p.transfers == 0
    assert_valid_equal(y1, reference(model, tok, lens), lens)


@pytest.mark.parametrize("seed", range(4))
def test_local_pipeline_ordering_and_correspondence(seed):
    """SPEC.md:714 (scaled): 48 batches with random B in [1,8], S in {4,8,16}, from 16 concurrent
    submitters, random delays injected in dispatch lanes and worker admission, pp = 4 -> every future
    holds ITS batch's oracle output, every stage ran keys 0,1,2,... in order, 3 transfers per batch,
    and no deadlock (watchdog)."""
    model = make_model()
    pp = 4
    trace = pl.Trace()
    runners = [OracleStage(model, a, b, i == 0, i == pp - 1) for i, (a, b) in enumerate(plan(SHAPE["L"], pp))]
    p = pl.LocalPipeline(runners, admit_delay=0.004, lane_delay=0.004, seed=seed, trace=trace)
    rng = random.Random(seed)
    batches = [random_batch(rng, 100 * seed + i) for i in range(48)]
    futs = [None] * len(batches)

    def submitter(idx):
        for i in idx:
            futs[i] = p.submit(*batches[i])

    ts = [threading.Thread(target=submitter, args=(list(range(j, 48, 16)),)) for j in range(16)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    outs = [f.result(timeout=60) for f in futs]
    p.shutdown(timeout=30)
    for (tok, lens), y in zip(batches, outs):
        assert_valid_equal(y, reference(model, tok, lens), lens)
    for s in range(pp):
        assert trace.keys(s) == list(range(48))
    admitted = [trace.keys(s, "admit") for s in range(pp)]
    assert any(a != sorted(a) for a in admitted), "the injected delays never reordered an admission"
    assert p.transfers == (pp - 1) * 48


def test_local_pipeline_stage_failure_fails_only_that_key():
    model = make_model()

    class Flaky(OracleStage):
        def __call__(self, cmd, x):
            if cmd.key == 1:
                raise ValueError("injected")
            return super().__call__(cmd, x)

    runners = [OracleStage(model, 0, 2, True, False), Flaky(model, 2, 4, False, True)]
    p = pl.LocalPipeline(runners, n_lanes=1)
    items = [(synth.tokens(2, 4, SHAPE["V"], [4, 2], i), [4, 2]) for i in range(3)]
    futs = [p.submit(*it) for it in items]
    assert_valid_equal(futs[0].result(30), reference(model, *items[0]), items[0][1])
    with pytest.raises(pl.StageFailed) as ei:
        futs[1].result(30)
    assert ei.value.key == 1 and ei.value.stage == 1
    assert_valid_equal(futs[2].result(30), reference(model, *items[2]), items[2][1])
    p.shutdown()


class SleepStage:
    def __init__(self, c):
        self.c = c

    def __call__(self, cmd, x):
        time.sleep(self.c)
        return torch.zeros(cmd.rows(), 1) if x is None else x


def test_local_pipeline_overlap_bound():
    """non-blocking overlap -- M batches through P stages of per-stage time c take
    <= (P + M - 1) c (1 + eps): pipeline fill + steady state, no blocking rendezvous."""
    c, P, M = 0.04, 4, 12
    p = pl.LocalPipeline([SleepStage(c) for _ in range(P)])
    t0 = time.monotonic()
    futs = [p.submit(np.zeros((1, 2), np.int32), [2]) for _ in range(M)]
    submitted = time.monotonic() - t0
    [f.result(30) for f in futs]
    elapsed = time.monotonic() - t0
    p.shutdown()
    assert submitted < c  # submit returns before any stage finishes
    assert elapsed <= (P + M - 1) * c * 1.25
    assert elapsed >= (P + M - 1) * c * 0.95


# ----------------------------------------------------------------------------- multi-process (gloo)
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dist_worker(rank, world, port, pp, tp, n_batches, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cmd_group = dist.new_group(backend="gloo")
        res_group = dist.new_group(backend="gloo")
        model = make_model()
        stage = rank // tp
        a, b = plan(SHAPE["L"], pp)[stage]
        trace = pl.Trace()
        H = SHAPE["H"]
        link = pl.DistLink(pp, tp, act_spec=lambda c: ((c.rows(), H), torch.float64, "cpu"),
                           out_spec=lambda c: ((c.batch, c.max_len, H), torch.float64, "cpu"),
                           cmd_group=cmd_group, act_group=None, res_group=res_group)
        runner = OracleStage(model, a, b, stage == 0, stage == pp - 1)
        worker = pl.StageWorker(stage, pp, runner, link, admit_delay=0.003, trace=trace, seed=rank).start()
        res = {}
        if rank == 0:
            engine = pl.Engine(link, 2 * pp, lane_delay=0.003, seed=7)
            link.engine = engine
            link.start_results()
            rng = random.Random(11)
            batches = [random_batch(rng, 500 + i) for i in range(n_batches)]
            futs = [engine.submit(*bt) for bt in batches]
            outs = [f.result(timeout=120) for f in futs]
            engine.shutdown()
            link.join_results(30)
            ok = True
            for (tok, lens), y in zip(batches, outs):
                ref = reference(model, tok, lens)
                for bb, n in enumerate(lens):
                    ok &= bool(np.array_equal(y.numpy()[bb, :n], ref[bb, :n])) and not np.any(y.numpy()[bb, n:])
            res["ok"] = ok
        worker.join(60)
        res.update(rank=rank, keys=trace.keys(stage), transfers=worker.transfers, calls=runner.calls,
                   error=repr(worker.error) if worker.error else None)
        dist.barrier()
        dist.destroy_process_group()
        q.put(res)
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put({"rank": rank, "exc": repr(e), "tb": traceback.format_exc()})


@pytest.mark.parametrize("pp,tp", [(3, 1), (2, 2)])
def test_dist_pipeline_gloo(pp, tp):
    """One process per (stage, TP rank) under torch.distributed: commands from the engine on rank 0,
    packed activations stage to stage, results back to rank 0; every stage runs keys 0..n-1 in order,
    pp - 1 transfers per batch per TP rank, every result = the oracle of its own batch."""
    world, n = pp * tp, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, pp, tp, n, q)) for r in range(world)]
    [p.start() for p in procs]
    res = [q.get(timeout=240) for _ in range(world)]
    [p.join(60) for p in procs]
    res = {r["rank"]: r for r in res}
    for r in range(world):
        assert "exc" not in res[r], res[r].get("tb")
        assert res[r]["error"] is None
        assert res[r]["keys"] == list(range(n))
        assert res[r]["calls"] == n
        stage = r // tp
        assert res[r]["transfers"] == (0 if stage == pp - 1 else n)
    assert res[0]["ok"]
