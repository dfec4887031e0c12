"""bench.py -- valid tokens/s and batch latency of the DRCE tensor-parallel GPT layer stack on B200.

Metric (BASELINE.json): "valid tokens/sec & batch latency, GPT-3-13B-shape stack, TP 1/2/4/8 B200".
One step = one forward pass of the whole hot path (index maps, embed+pack,
40 x (LN, QKV GEMM, unpack, attention, repack, out-proj GEMM, [allreduce], residual+LN, up GEMM,
down GEMM, [allreduce], residual+LN), final LN + unpack) over one synthetic batch of the GPT-3-13B
shape (B=16, max_len=512, exact padding ratio 0.5 -> T=4096 valid tokens), bf16, random-init weights.

  python bench.py [--gpus N --steps K --warmup W]       energon arm (N>1: under torchrun, TP=N)
      --comm nccl|p2p     TP exchange: NCCL, or the fused peer-memory kernels (CUDA IPC)
      --pp P              NBPP: one pipeline stage per rank (world == P), --pp-batches in flight
      --local-tp k        TP=k per-rank shapes emulated on ONE GPU (in-device reductions)
      --config / --p / --regime / --layers / --graph / --drce    workload and option overrides
  python bench.py --impl reference ...                  the fp64 CPU oracle arm (rank 0 only)

Timing: W untimed warm-up steps, then K steps bracketed by barrier + cuda.synchronize, CUDA events
on the forward stream, max over ranks.  value = valid tokens per step * K / time (TP: every rank
works on the same batch, so the job's units are the batch's T valid tokens -> "scaling": "strong").
The per-step working set (25 GB of bf16 weights at TP=1) is far larger than the 126 MB L2, so no
explicit flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "valid tokens/sec & batch latency, GPT-3-13B-shape stack, TP 1/2/4/8 B200"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="energon", choices=["energon", "reference"])
    ap.add_argument("--config", default="gpt3_13b")
    ap.add_argument("--p", type=float, default=None, help="padding ratio (exact-p configs)")
    ap.add_argument("--regime", default=None, choices=[None, "exact_p", "paper", "random"])
    ap.add_argument("--seed", type=int, default=0, help="first seed of the rotated batches")
    ap.add_argument("--seeds", type=int, default=5,
                    help="SURVEY.md 8(d): the timed steps rotate over the batches of seeds seed..seed+seeds-1 "
                         "(new lengths and tokens every step); per-seed medians are reported")
    ap.add_argument("--drce", type=int, default=1)
    ap.add_argument("--ln-fuse", type=int, default=0,
                    help="N3 (TP = 1, bf16): LN1 / LN2 applied in the QKV / MLP-up GEMM prologues (ENERGON_OPT_LN_FUSE)")
    ap.add_argument("--layers", type=int, default=None, help="override the layer count (debug only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tp-check", action="store_true",
                    help="skip the post-timing TP = k checks (replicas bit-identical, TP = k vs TP = 1 on rank 0)")
    ap.add_argument("--no-ab", action="store_true", help="skip the DRCE-off (padded) A/B")
    ap.add_argument("--graph", type=int, default=None,
                    help="replay each forward as a CUDA graph (ENERGON_OPT_GRAPH); default on for one GPU, off "
                         "under torchrun (NCCL collectives run eagerly)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pp", type=int, default=1,
                    help="NBPP: one pipeline stage per rank (torchrun, world == pp), --pp-batches batches in flight")
    ap.add_argument("--pp-batches", type=int, default=8)
    ap.add_argument("--comm", default="p2p", choices=["nccl", "p2p"],
                    help="TP exchange for N > 1: the fused peer-memory kernels over CUDA IPC (default; the exchange "
                         "the multi-process GPU tests check against the oracle) or NCCL")
    ap.add_argument("--local-tp", type=int, default=0,
                    help="emulate TP=k on ONE GPU with a local group (ranks serialised; per-rank kernel "
                         "shapes and ncu evidence of TP=k, not a TP=k latency)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ============================================================================= oracle (CPU) arm
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def step_flops(H, L, lens) -> float:
    """Algorithmic FLOPs of one DRCE forward: per sequence of n valid tokens and per layer,
    linears 24 H^2 n and causal attention 2 H n (n + 1) (QK^T and PV over the n(n+1)/2 allowed pairs)."""
    return float(L) * sum(24.0 * H * H * n + 2.0 * H * n * (n + 1) for n in lens)


def oracle_sample(args, shape, lens, tok):
    """SURVEY.md 8(d) "Oracle timing": one layer (layer 0) of the fp64 oracle over the LONGEST and the
    SHORTEST sequence of the batch, each at its full length (exact sub-problems by sequence independence,
    P12), measured, then extrapolated to the whole step (all sequences, all layers) by the FLOP ratio of
    step_flops.  Returns (run, describe): run() -> sample seconds; describe(t) -> (tokens/s, note)."""
    import numpy as np

    import oracle
    import synth
    H, L = shape["H"], shape["L"]
    picks = sorted({int(np.argmax(lens)), int(np.argmin(lens))})
    layers, emb = synth.model_host(1, H, shape["F"], shape["V"], shape["max_seq"], args.seed, True, layer_ids=[0])
    cfg = oracle.make_cfg(1, H, shape["h"], shape["F"])
    xs = [(oracle.embed(cfg, emb, tok[b:b + 1, :lens[b]]), lens[b]) for b in picks]
    f_sample = step_flops(H, 1, [n for _, n in xs])
    f_step = step_flops(H, L, lens)
    T = sum(lens)

    def run():
        t0 = time.perf_counter()
        for X, n in xs:
            oracle.layers_padded(cfg, layers, 0, 1, X, [n])
        return time.perf_counter() - t0

    def describe(t):
        est = t * f_step / f_sample
        note = (f"fp64 oracle (oracle/oracle.c, OpenMP), layer 0 of {L} over the longest ({max(lens)}) and the "
                f"shortest ({min(lens)}) sequence at full length ({t:.1f} s for {f_sample / 1e9:.0f} GFLOP), "
                f"extrapolated by the FLOP ratio {f_step / f_sample:.0f}x to the whole step (T={T}, {L} layers): "
                f"{est:.0f} s per step, extrapolated; CPU: {cpu_model()}, {oracle.num_threads()} OpenMP threads")
        return T / est, note

    return run, describe


def reference_arm(args, world, rank):
    if rank != 0:
        return  # rank 0 alone runs the oracle arm
    import oracle
    import synth
    shape = dict(synth.SHAPES[args.config])
    if args.layers:
        shape["L"] = args.layers
    bcfg = synth.BATCHES[args.config]
    lens = synth.batch_lengths(args.config, args.seed, p=args.p, regime=args.regime)
    tok = synth.tokens(bcfg["B"], bcfg["S"], shape["V"], lens, args.seed)
    run, describe = oracle_sample(args, shape, lens, tok)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    t = sum(times) / len(times)
    value, note = describe(t)
    step_s = sum(lens) / value
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s, "sample_s_per_step": t,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": workload_config(args, shape, bcfg, lens, world),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                            "sample": note, "cpu_model": cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def workload_config(args, shape, bcfg, lens, world):
    T = sum(lens)
    B, S = bcfg["B"], bcfg["S"]
    return {"workload": f"{args.config}: {shape['L']} layers, H={shape['H']}, {shape['h']} heads, B={B}, "
                        f"max_len={S}, padding {1 - T / (B * S):.3f} (T={T}), bf16, TP={world}",
            "layers": shape["L"], "hidden": shape["H"], "heads": shape["h"], "batch": B, "max_len": S,
            "padding_ratio": round(1 - T / (B * S), 4), "valid_tokens_per_step": T, "tp": world,
            "parallelism": f"tp{world}", "drce": bool(args.drce), "cuda_graph": bool(getattr(args, "graph", 0)),
            "tp_exchange": (getattr(args, "comm", "nccl") if world > 1 else "none"),
            "l2": "no flush: per-step working set (weights) > 126 MB L2"}


# ============================================================================= energon (GPU) arm
class Engine:
    """One rank's context, or a local group of k contexts on this GPU (--local-tp)."""

    def __init__(self, energon, ctxs):
        self.e, self.ctxs = energon, ctxs

    def forward(self, tok, lens, out, stream):
        if len(self.ctxs) == 1:
            self.e.energon_forward(self.ctxs[0], tok, lens, out, stream)
        else:
            self.e.energon_forward_group(self.ctxs, tok, lens, out, stream)

    def set_option(self, opt, v):
        for c in self.ctxs:
            self.e.energon_set_option(c, opt, v)

    def set_profiling(self, on):
        for c in self.ctxs:
            self.e.energon_set_profiling(c, on)

    def profile(self):
        tot = {}
        for c in self.ctxs:
            for k, v in self.e.energon_get_profile(c).items():
                tot[k] = tot.get(k, 0) + v
        return tot

    def launches(self):
        return sum(self.e.energon_get_stats(c)["kernel_launches"] for c in self.ctxs)

    def sync(self):
        self.e.energon_sync(self.ctxs[0])

    def destroy(self):
        for c in self.ctxs:
            self.e.energon_destroy(c)


def _vs_tp1(args, energon, out, bt, shape, B, S):
    """Rank 0 of a TP = k run: the same batch through a TP = 1 context of the same weights on this GPU;
    max-abs-rel of the TP = k output `out` against it over the valid positions."""
    import torch
    import synth
    H, L = shape["H"], shape["L"]
    cfg1 = energon.make_config(L, H, shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S, dtype="bf16",
                               drce=args.drce, tp_size=1, tp_rank=0, device=torch.cuda.current_device())
    c1 = energon.energon_init(cfg1, None)
    try:
        emb = {n: synth.emb_tensor_device(n, H, shape["V"], shape["max_seq"], args.seed, True, torch.bfloat16)
               for n in synth.EMB_TENSORS}
        energon.energon_load_embeddings(c1, emb["tok_emb"], emb["pos_emb"], emb["lnf_g"], emb["lnf_b"])
        del emb
        for l in range(L):
            w = {n: synth.layer_tensor_device(n, l, H, shape["F"], args.seed, True, torch.bfloat16)
                 for n in synth.LAYER_TENSORS}
            energon.energon_load_layer_weights(c1, l, w)
            del w
        out1 = torch.empty_like(out)
        energon.energon_forward(c1, bt["tok_d"], bt["lens"], out1, torch.cuda.current_stream())
        energon.energon_sync(c1)
        torch.cuda.synchronize()
        num = den = 0.0
        for b, n in enumerate(bt["lens"]):
            y, y1 = out[b, :n].float(), out1[b, :n].float()
            num = max(num, (y - y1).abs().max().item())
            den = max(den, y1.abs().max().item())
        return {"max_abs_rel_vs_tp1": num / den}
    finally:
        energon.energon_destroy(c1)
        torch.cuda.empty_cache()


def tp_check(args, energon, eng, fwd, out, bt, shape, B, S, world, rank, dist, barrier, plumb):
    """After the timed region of a TP = k run (k ranks, or a --local-tp group): (1) every rank's output of the
    first batch is bit-identical (replicas: each packed row is reduced once, by its owner, and
    every rank receives the same LayerNorm rows); (2) rank 0 runs the same batch through a TP = 1 context of
    the same weights on its own GPU and reports max-abs-rel of the TP = k output against it
    over the valid positions -- the north star's "TP = k equals TP = 1" property, measured over the real
    exchange.  Not timed."""
    import hashlib
    import torch
    fwd(0)
    eng.sync()
    torch.cuda.synchronize()
    digest = hashlib.sha256(out.view(torch.int16).cpu().numpy().tobytes()).hexdigest()
    res = {"batch_seed": bt["seed"], "bar": 2e-2}
    if dist is not None:
        digs = [None] * world
        dist.all_gather_object(digs, digest)
        res["replicas_bit_identical"] = len(set(digs)) == 1
    H, L = shape["H"], shape["L"]
    full_bytes = 2 * (12 * H * H + 13 * H) * L + 2 * (shape["V"] + shape["max_seq"]) * H
    if full_bytes > 100e9:
        res["vs_tp1"] = f"skipped: a TP=1 copy ({full_bytes / 1e9:.0f} GB) does not fit next to the shard"
        barrier()
        return res
    if rank == 0:
        try:
            res.update(_vs_tp1(args, energon, out, bt, shape, B, S))
            res["pass"] = res["max_abs_rel_vs_tp1"] <= res["bar"] and res.get("replicas_bit_identical", True)
        except Exception as e:  # noqa: BLE001 -- reported; the other ranks are waiting at the barrier below
            res["vs_tp1"] = f"error: {type(e).__name__}: {str(e)[:200]}"
    barrier()
    return res


def energon_arm(args, world, rank, local):
    import numpy as np
    import torch

    import synth
    from paper_2209_02341_b200 import energon

    # ENERGON_BENCH_SHARE_GPU=1 (test hook): every rank on cuda:0 with gloo plumbing and the P2P exchange
    # (NCCL refuses two ranks on one GPU) -- exercises the N > 1 bench path on a single-GPU box; its
    # timings mean nothing (the ranks time-slice one GPU)
    share = os.environ.get("ENERGON_BENCH_SHARE_GPU") == "1" and world > 1
    if share:
        local = 0
        args.comm = "p2p"
    torch.cuda.set_device(local)
    plumb = "cpu" if share else "cuda"
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    energon.load_library()
    shape = dict(synth.SHAPES[args.config])
    if args.layers:
        shape["L"] = args.layers
    bcfg = synth.BATCHES[args.config]
    B, S = bcfg["B"], bcfg["S"]
    H = shape["H"]
    # the rotated batches (SURVEY.md 8(d) "Seeds 0-4"): lengths + tokens of seeds seed .. seed+seeds-1;
    # with exact-p lengths every batch has the same T but a different length mix
    seeds = [args.seed + i for i in range(max(1, args.seeds))]
    batches = []
    for sd in seeds:
        lens = synth.batch_lengths(args.config, sd, p=args.p, regime=args.regime)
        batches.append({"seed": sd, "lens": lens, "T": sum(lens), "tok": synth.tokens(B, S, shape["V"], lens, sd)})
    lens0 = batches[0]["lens"]

    comm = energon.COMM_P2P if (args.comm == "p2p" and world > 1) else energon.COMM_NCCL
    cfg = energon.make_config(shape["L"], H, shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S,
                              dtype="bf16", drce=args.drce, tp_size=world, tp_rank=rank, device=local, comm=comm)
    uid = None
    if world > 1:
        from paper_2209_02341_b200 import dist as edist
        if comm == energon.COMM_NCCL:
            uid = edist.broadcast_bytes(energon.energon_get_unique_id() if rank == 0 else None, 128, device=plumb)
        for bt in batches:  # the engine command's seq_lens: rank 0's list on every rank
            bt["lens"] = edist.broadcast_lengths(bt["lens"], device=plumb)
    if args.local_tp > 1:
        ctxs = energon.energon_init_local_group(cfg, args.local_tp)
    else:
        ctxs = [energon.energon_init(cfg, uid)]
    p2p_fallback = None
    if comm == energon.COMM_P2P and world > 1:  # map every rank's exchange region (CUDA IPC handles, all-gathered)
        err = ""
        try:
            handles = [None] * world
            dist.all_gather_object(handles, energon.energon_p2p_handle(ctxs[0]))
            energon.energon_p2p_connect(ctxs[0], handles)
        except energon.EnergonError as e:  # peer mapping refused on this box: every rank falls back to NCCL
            err = str(e)
        errs = [None] * world
        dist.all_gather_object(errs, err)
        bad = [e for e in errs if e]
        if bad and not share:
            energon.energon_destroy(ctxs[0])
            comm = energon.COMM_NCCL
            args.comm = "nccl"
            cfg = energon.make_config(shape["L"], H, shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S,
                                      dtype="bf16", drce=args.drce, tp_size=world, tp_rank=rank, device=local,
                                      comm=comm)
            uid = edist.broadcast_bytes(energon.energon_get_unique_id() if rank == 0 else None, 128, device=plumb)
            ctxs = [energon.energon_init(cfg, uid)]
            p2p_fallback = f"p2p connect failed ({bad[0][:160]}); NCCL exchange used"
        elif bad:
            raise RuntimeError(bad[0])
    eng = Engine(energon, ctxs)

    # weights: generated on the device by the seeded counter-based generator, loaded unsharded
    emb = {n: synth.emb_tensor_device(n, H, shape["V"], shape["max_seq"], args.seed, True, torch.bfloat16)
           for n in synth.EMB_TENSORS}
    for c in ctxs:
        energon.energon_load_embeddings(c, emb["tok_emb"], emb["pos_emb"], emb["lnf_g"], emb["lnf_b"])
    del emb
    for l in range(shape["L"]):
        w = {n: synth.layer_tensor_device(n, l, H, shape["F"], args.seed, True, torch.bfloat16)
             for n in synth.LAYER_TENSORS}
        for c in ctxs:
            energon.energon_load_layer_weights(c, l, w)
        del w
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if args.graph is None:
        args.graph = 1 if world == 1 else 0
    eng.set_option(energon.OPT_GRAPH, args.graph)
    if args.ln_fuse:
        eng.set_option(energon.OPT_LN_FUSE, 1)

    stream = torch.cuda.current_stream()
    for bt in batches:
        bt["tok_d"] = torch.from_numpy(bt["tok"]).cuda()
    out = torch.empty(B, S, H, dtype=torch.bfloat16, device="cuda")
    nb = len(batches)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        from paper_2209_02341_b200 import dist as edist
        return edist.max_over_ranks(x, device=plumb)

    def fwd(i, tok=None, o=None):
        bt = batches[i % nb]
        eng.forward(bt["tok_d"] if tok is None else tok, bt["lens"], out if o is None else o, stream)

    # warm-up: W steps, and at least one per rotated batch (each batch's first forward records its graph)
    warm = max(args.warmup, nb)
    for i in range(warm):
        fwd(i)
    eng.sync()

    # ---------------- device-timed region: inputs resident in HBM (no per-launch instrumentation)
    launches0 = eng.launches()
    clocks = ClockSampler(local)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    prof_range = os.environ.get("ENERGON_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if prof_range:
        torch.cuda.cudart().cudaProfilerStart()
    evs[0].record(stream)
    for i in range(args.steps):
        fwd(i)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    if prof_range:
        torch.cuda.cudart().cudaProfilerStop()
    barrier()
    clk = clocks.stop()
    eng.sync()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = max_over_ranks(evs[0].elapsed_time(evs[-1]))
    launches = eng.launches() - launches0
    tokens_timed = sum(batches[i % nb]["T"] for i in range(args.steps))
    value = tokens_timed / (total_ms * 1e-3)
    per_seed = {}
    for i, ms in enumerate(step_ms):
        per_seed.setdefault(batches[i % nb]["seed"], []).append(ms)
    seed_ms = {sd: statistics.median(v) for sd, v in per_seed.items()}
    seed_tok_s = {sd: batches[[b["seed"] for b in batches].index(sd)]["T"] / (ms * 1e-3) for sd, ms in seed_ms.items()}

    # ---------------- instrumented pass: the same K steps with CUDA events around every launch on
    # the forward stream (energon_set_profiling) -> per-kernel-class device time for the roofline
    eng.set_profiling(True)
    barrier()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for i in range(args.steps):
        fwd(i)
    p1.record(stream)
    torch.cuda.synchronize()
    barrier()
    prof = eng.profile()
    prof_ms = p0.elapsed_time(p1) / args.steps
    eng.set_profiling(False)

    # ---------------- end-to-end: host tokens -> device, forward, result -> host, every step.  The
    # device->host copy of step i's result runs on a copy stream while step i+1 computes (two device
    # output buffers, two pinned host buffers); the timed region ends after the last copy has landed.
    e2e = None
    if not args.no_e2e:
        toks_h = [torch.from_numpy(bt["tok"]).pin_memory() for bt in batches]
        outs = [out, torch.empty_like(out)]
        outs_h = [torch.empty(B, S, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        copy_st = torch.cuda.Stream()
        done = [torch.cuda.Event(), torch.cuda.Event()]  # buffer i's D2H finished
        ready = [torch.cuda.Event(), torch.cuda.Event()]  # buffer i's forward finished

        def e2e_step(i):
            k = i & 1
            stream.wait_event(done[k])  # the D2H of step i-2 has read outs[k]
            tok_d = batches[i % nb]["tok_d"]
            tok_d.copy_(toks_h[i % nb], non_blocking=True)  # this step's tokens, host -> device
            fwd(i, tok_d, outs[k])
            ready[k].record(stream)
            copy_st.wait_event(ready[k])
            with torch.cuda.stream(copy_st):
                outs_h[k].copy_(outs[k], non_blocking=True)
            done[k].record(copy_st)

        for k in range(2):
            done[k].record(copy_st)
        for i in range(nb if nb % 2 == 0 else 2 * nb):  # every (batch, output buffer) pair records its graph
            e2e_step(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.steps):
            e2e_step(i)
        stream.wait_event(done[(args.steps - 1) & 1])  # the last result is on the host
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": tokens_timed / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": toks_h[0].numel() * 4,
               "d2h_bytes_per_step": outs_h[0].numel() * 2, "ms_per_step": e2e_ms / args.steps,
               "overlap": "step i's device->host copy overlaps step i+1 (copy stream, double-buffered output)"}
    eng.sync()

    # ---------------- DRCE A/B: the first batch with the linears on all B*S padded rows
    drce_ab = None
    T0 = batches[0]["T"]
    if not args.no_ab and args.drce:
        eng.set_option(energon.OPT_DRCE, 0)
        fwd(0)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nab = max(2, args.steps // 2)
        barrier()
        torch.cuda.synchronize()
        a0.record(stream)
        for _ in range(nab):
            fwd(0)
        a1.record(stream)
        torch.cuda.synchronize()
        barrier()
        off_ms = max_over_ranks(a0.elapsed_time(a1)) / nab
        eng.set_option(energon.OPT_DRCE, 1)
        fwd(0)
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(nab):
            fwd(0)
        b1.record(stream)
        torch.cuda.synchronize()
        barrier()
        on_ms = max_over_ranks(b0.elapsed_time(b1)) / nab
        drce_ab = {"batch_seed": batches[0]["seed"], "drce_on_ms": on_ms, "drce_off_ms": off_ms,
                   "latency_reduction": 1 - on_ms / off_ms, "valid_tok_s_off": T0 / (off_ms * 1e-3),
                   "padding_ratio": 1 - T0 / (B * S), "ideal_reduction": 1 - T0 / (B * S),
                   "note": "paper: up to 46.8% latency reduction at p=0.5 on A100 (PAPER.md:567-579)"}
    eng.sync()

    pk = peaks()
    gemm_ms_avg = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
    achieved = prof["gemm_flops"] / (prof["gemm_ms"] * 1e-3) / 1e12 if prof["gemm_ms"] > 0 else None
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "gemm_traffic.json")))
        traffic = tr.get(args.config, {}).get(f"tp{world}")
    except Exception:
        pass
    roofline = {"bound": "tensor", "kernel": "gemm_tc2_kernel (a4/a8/a10/a11, tcgen05 bf16)",
                "achieved": achieved, "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": (achieved / pk["bf16_tflops_sustained"]) if achieved else None, "traffic": traffic,
                "peak_source": f"{pk['source']} bf16_tflops_sustained (kernel timed inside a long step)",
                "frac_of_burst": (achieved / pk["bf16_tflops"]) if achieved else None,
                "frac_of_2250_nominal": (achieved / 2250.0) if achieved else None,
                "avg_launch_ms": gemm_ms_avg, "flops_per_step": prof["gemm_flops"] / args.steps,
                "share_of_step": prof["gemm_ms"] / args.steps / prof_ms,
                "measured_in": "instrumented pass of the same K steps (CUDA events around every launch)"}
    k_tp = world if args.local_tp <= 1 else args.local_tp
    exch_calls = prof["comm_calls"] / args.steps
    exchange = None
    if k_tp > 1:
        # allreduce-equivalent bus bandwidth of the 2 L exchanges per step (nccl-tests convention:
        # busbw = payload * 2 (k-1) / k / time), payload = the packed [T, H] bf16 partial
        payload = tokens_timed / args.steps * H * 2
        n_ex = 2 * shape["L"]
        ms = prof["comm_ms"] / args.steps
        exchange = {"kind": "local group (in-device)" if args.local_tp > 1 else args.comm, "exchanges_per_step": n_ex,
                    "payload_bytes": payload, "ms_per_step": ms,
                    "bus_gbs": (n_ex * payload * 2 * (k_tp - 1) / k_tp / (ms * 1e-3) / 1e9) if ms else None,
                    "launch_records_per_step": exch_calls,
                    "note": "time of the exchange launches (P2P: flag + reduce/LN + flag kernels, which also do the "
                            "bias + residual + LN2 work; NCCL: reduce-scatter + all-gather); nvlink peak 900 GB/s"}
    phases = {
        "gemm": {"ms_per_step": prof["gemm_ms"] / args.steps, "launches": prof["gemm_launches"] // args.steps,
                 "tflops": achieved},
        "attention": {"ms_per_step": prof["attn_ms"] / args.steps,
                      "tflops": prof["attn_flops"] / (prof["attn_ms"] * 1e-3) / 1e12 if prof["attn_ms"] else None},
        "memory_bound": {"ms_per_step": prof["mem_ms"] / args.steps,
                         "gbs": prof["mem_bytes"] / (prof["mem_ms"] * 1e-3) / 1e9 if prof["mem_ms"] else None,
                         "frac_of_hbm": (prof["mem_bytes"] / (prof["mem_ms"] * 1e-3) / 1e9 / pk["hbm_gbs"])
                         if prof["mem_ms"] else None},
        "exchange": {"ms_per_step": prof["comm_ms"] / args.steps, "calls": prof["comm_calls"] // args.steps},
        "note": "per-launch CUDA events (instrumented pass) add a few us to every launch and break the "
                "programmatic-launch overlap, which inflates the short memory-bound kernels most: the ncu "
                "launch list (profiles/) times residual+LN at ~42.5 us = ~5.9 TB/s of algorithmic traffic",
    }
    gpus_active = world if not share else 1
    config = workload_config(args, shape, bcfg, lens0, k_tp)
    config["seeds"] = seeds
    if args.ln_fuse:
        config["ln_fuse"] = True
    if p2p_fallback:
        config["p2p_fallback"] = p2p_fallback
    config["valid_tokens_per_step"] = tokens_timed / args.steps
    result = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "warmup_steps_run": warm, "ms_per_step": total_ms / args.steps,
              "latency_ms_p50": statistics.median(step_ms), "latency_ms_p95": sorted(step_ms)[
                  min(len(step_ms) - 1, int(round(0.95 * (len(step_ms) - 1))))],
              "per_seed": {"ms_median": {str(k): v for k, v in seed_ms.items()},
                           "tok_s": {str(k): v for k, v in seed_tok_s.items()},
                           "median_tok_s": statistics.median(seed_tok_s.values())},
              "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
              "data": "synthetic (seeded counter-based generator; random-init weights of the GPT-3-13B shape; "
                      f"batches of seeds {seeds[0]}..{seeds[-1]} rotated step by step)",
              "config": config, "clocks": clk, "e2e": e2e, "gpus_active": gpus_active,
              "gpu_launches": int(launches), "roofline": roofline, "phases": phases, "exchange": exchange,
              "drce_ab": drce_ab}

    if rank == 0 and world == 1 and args.local_tp <= 1 and not args.no_cpu_baseline:
        import oracle
        run, describe = oracle_sample(args, shape, batches[0]["lens"], batches[0]["tok"])
        v, note = describe(run())
        result["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                                  "sample": note, "cpu_model": cpu_model()}
    if k_tp > 1 and not args.no_tp_check:
        # never let the (untimed) check cost the measured line: errors are reported, every rank still meets the
        # barriers inside tp_check
        try:
            result["tp_check"] = tp_check(args, energon, eng, fwd, out, batches[0], shape, B, S, world, rank, dist,
                                          barrier, plumb)
        except Exception as e:  # noqa: BLE001
            result["tp_check"] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    if args.local_tp > 1:
        result["local_tp_emulation"] = (f"TP={args.local_tp} ranks run serially on ONE GPU (in-device reductions): "
                                        "per-rank kernel shapes of TP=k, not a TP=k latency")
    if share:
        result["shared_gpu"] = "ENERGON_BENCH_SHARE_GPU=1: all ranks time-slice cuda:0 -- the timings mean nothing"
    if rank == 0:
        print(json.dumps(result), flush=True)
    eng.destroy()
    if dist is not None:
        dist.destroy_process_group()


# ============================================================================= NBPP pipeline arm
def pipeline_arm(args, world, rank, local):
    """Non-blocking pipeline parallelism: rank i runs stage i (a contiguous layer
    range, energon_forward_stage), the engine on rank 0 submits --pp-batches batches of the workload at
    once; value = valid tokens of all batches / device-clock time from the first submit to the last
    result (max over ranks).  One process per GPU, activations rank to rank over NCCL (or through host
    memory with ENERGON_BENCH_SHARE_GPU=1, where the timing is meaningless)."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2209_02341_b200 import energon
    from paper_2209_02341_b200 import pipeline as pl

    share = os.environ.get("ENERGON_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cmd_group = dist.new_group(backend="gloo")
    res_group = dist.new_group(backend="gloo" if share else "nccl")
    energon.load_library()
    shape = dict(synth.SHAPES[args.config])
    if args.layers:
        shape["L"] = args.layers
    bcfg = synth.BATCHES[args.config]
    B, S = bcfg["B"], bcfg["S"]
    H = shape["H"]
    lens = synth.batch_lengths(args.config, args.seed, p=args.p, regime=args.regime)
    T = sum(lens)
    tok_np = synth.tokens(B, S, shape["V"], lens, args.seed)
    l0, l1 = energon.energon_stage_plan(shape["L"], world)[rank]
    cfg = energon.make_config(shape["L"], H, shape["h"], shape["F"], shape["V"], shape["max_seq"], B * S,
                              dtype="bf16", drce=args.drce, device=local)
    ctx = energon.energon_init(cfg)
    if rank == 0 or rank == world - 1:
        emb = {n: synth.emb_tensor_device(n, H, shape["V"], shape["max_seq"], args.seed, True, torch.bfloat16)
               for n in synth.EMB_TENSORS}
        energon.energon_load_embeddings(ctx, emb["tok_emb"], emb["pos_emb"], emb["lnf_g"], emb["lnf_b"])
        del emb
    for l in range(l0, l1):
        w = {n: synth.layer_tensor_device(n, l, H, shape["F"], args.seed, True, torch.bfloat16)
             for n in synth.LAYER_TENSORS}
        energon.energon_load_layer_weights(ctx, l, w)
        del w
    torch.cuda.synchronize()
    dev = f"cuda:{local}"
    link = pl.DistLink(world, 1, act_spec=lambda c: ((c.rows(bool(args.drce)), H), torch.float32, dev),
                       out_spec=lambda c: ((c.batch, c.max_len, H), torch.bfloat16, dev),
                       cmd_group=cmd_group, act_group=None, res_group=res_group, stage_via_host=share)
    runner = pl.EnergonStageRunner(ctx, l0, l1, first=rank == 0, last=rank == world - 1, hidden=H,
                                   out_dtype=torch.bfloat16, device=local, drce=bool(args.drce))
    worker = pl.StageWorker(rank, world, runner, link).start()
    engine = None
    if rank == 0:
        engine = pl.Engine(link, 2 * world)
        link.engine = engine
        link.start_results()

    def run_round(n):
        futs = [engine.submit(tok_np, lens) for _ in range(n)]
        for f in futs:
            f.result(timeout=600)

    # warm-up: every stage compiles its launch path; then the timed round (rank 0 drives)
    if rank == 0:
        run_round(max(args.warmup, 1))
    dist.barrier(group=cmd_group)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if rank == 0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_round(args.pp_batches)
        e1.record()
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1)
    dist.barrier(group=cmd_group)
    wall_ms = (time.perf_counter() - t0) * 1e3
    if rank == 0:
        engine.shutdown()
        link.join_results(60)
    worker.join(120)
    t = torch.tensor([wall_ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=cmd_group)
    if rank == 0:
        ms = max(dev_ms, 0.0)
        tokens = T * args.pp_batches
        print(json.dumps({
            "metric": METRIC, "value": tokens / ms * 1e3, "unit": "tokens/s", "n_gpus": world,
            "steps": args.pp_batches, "warmup": max(args.warmup, 1), "ms_per_step": ms / args.pp_batches,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter-based generator; random-init weights)",
            "config": dict(workload_config(args, shape, bcfg, lens, 1), parallelism=f"pp{world}",
                           pipeline={"stages": world, "batches_in_flight": args.pp_batches,
                                     "stage_layers": energon.energon_stage_plan(shape["L"], world),
                                     "transfers_per_batch": world - 1,
                                     "activation_transport": "host (shared GPU)" if share else "nccl p2p"}),
            "wall_ms_max_over_ranks": float(t.item()),
            "note": "NBPP: engine + distributed consistency queue (pipeline.py); value = valid tokens of all "
                    "batches / time from the first submit to the last result on rank 0's clock"}))
    energon.energon_destroy(ctx)
    dist.destroy_process_group()


def self_launch(args) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: relaunch this script under torch.distributed.run, one
    rank per GPU on this node (rendezvous on 127.0.0.1), with the same arguments; rank 0 prints the line."""
    import socket
    if os.environ.get("ENERGON_BENCH_SHARE_GPU") != "1" and args.impl != "reference":
        try:
            import torch
            n = torch.cuda.device_count()
        except Exception:
            n = 0
        if n < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {n} "
                                                         "(ENERGON_BENCH_SHARE_GPU=1 runs every rank on cuda:0)"}),
                  flush=True)
            return 2
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, ENERGON_BENCH_SELF_LAUNCHED="1")
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(self_launch(args))
    if args.gpus > 1 and world != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if world > 1:
        # the driver reads NCCL's own log (comm_nranks) to confirm the group spans every GPU
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        reference_arm(args, world, rank)
    elif args.pp > 1:
        if args.pp != world:
            print(json.dumps({"error": "--pp P needs exactly P ranks (one stage per GPU)"}))
            sys.exit(2)
        pipeline_arm(args, world, rank, local)
    else:
        energon_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
