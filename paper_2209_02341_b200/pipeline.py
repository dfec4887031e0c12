"""Non-blocking pipeline parallelism (NBPP, sec 4.2 / fig:engine) and the engine
front-end: the CONTROL PLANE around the C-ABI stage entry
``energon_forward_stage`` (include/energon.h).  No arithmetic of the method lives here -- every layer
runs in libenergon.so; this module only orders batches, moves activation buffers between stages and
hands results back.

The paper's two designs, restated:

* "a thread pool in the engine that fetches batches from the batch list.  For a single thread in the
  engine, it will launch an inference task to workers with input tensor and some meta information"
  (PAPER.md:328-330): ``Engine`` -- ``submit`` returns a future immediately; a pool of dispatch lanes
  takes the unique key from the engine's ``LoopCounter`` and sends the ``Command`` (seq_lens always,
  tokens to the first stage) to every worker.
* "a distributed consistency queue ... a loop data structure that increments unidirectionally ... the
  worker will add the batch into the local queue and use the remote unique value as a key ... the
  thread that acquires the lock ... takes the local unique key from the local loop data structure,
  find the batch uses the local key, and executes the batch":
  ``ConsistencyQueue`` -- commands may be admitted by several worker threads in any order; the compute
  thread always executes the next key of its own counter, so every stage processes keys 0, 1, 2, ...
  and the point-to-point activation transfers between consecutive stages (one per batch per link,
  "only (#GPU - 1) communications") match without tags even though batch and padding
  sizes differ from batch to batch (the deadlock the paper describes).

Two transports share the same ``StageWorker`` / ``Engine`` code:

* ``LocalPipeline`` -- every stage is a thread of this process (stages on one GPU, each on its own
  CUDA stream, hand-offs ordered by CUDA events; or the CPU for tests).
* ``DistLink`` -- one process per (stage, TP rank) under ``torch.distributed`` (rank = stage * tp +
  tp_rank, engine on rank 0): commands over a gloo group, activations over point-to-point sends on the
  default group (NCCL over NVLink on B200 boxes), results to rank 0 over their own group.

Readings: keys are unbounded 64-bit (the paper's "loop" is never said to wrap,
SPEC.md:427); with DRCE the activations travel packed ([T, H] fp32 rows); a stage failure
fails that key's result and the pipeline continues (the paper is silent).
"""
from __future__ import annotations

import queue
import random
import threading
import time
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass, field


class ProtocolError(RuntimeError):
    pass


class Closed(Exception):
    pass


class LoopCounter:
    """"a loop data structure that increments unidirectionally": 0, 1, 2, ..."""

    def __init__(self, start: int = 0):
        self._v = start
        self._lock = threading.Lock()

    def next(self) -> int:
        with self._lock:
            v = self._v
            self._v += 1
            return v

    def peek(self) -> int:
        with self._lock:
            return self._v


class ConsistencyQueue:
    """Per-worker queue keyed by the engine's unique keys.  ``pop_next`` returns the
    entry whose key equals the local counter and then increments it, whatever order the entries were
    inserted in; it blocks until that key arrives.  Inserts never block: a bound on pending entries
    would let a finite pool of admitting threads all wait behind later keys while the key the consumer
    needs sits in their backlog -- the very deadlock the queue exists to remove."""

    def __init__(self):
        self._items: dict[int, object] = {}
        self._next = LoopCounter()
        self._want = 0
        self._cv = threading.Condition()
        self._closed = False

    def insert(self, key: int, item) -> None:
        with self._cv:
            if key < self._want or key in self._items:
                raise ProtocolError(f"duplicate or stale key {key}")
            self._items[key] = item
            self._cv.notify_all()

    def pop_next(self, timeout: float | None = None):
        deadline = None if timeout is None else time.monotonic() + timeout
        with self._cv:
            while self._want not in self._items:
                if self._closed:
                    raise Closed()
                rem = None if deadline is None else deadline - time.monotonic()
                if rem is not None and rem <= 0:
                    raise TimeoutError(f"key {self._want} did not arrive")
                self._cv.wait(rem)
            key = self._next.next()
            assert key == self._want
            self._want += 1
            item = self._items.pop(key)
            self._cv.notify_all()
            return key, item

    def close(self) -> None:
        """No more inserts: pending keys are still popped in order, then pop_next raises Closed."""
        with self._cv:
            self._closed = True
            self._cv.notify_all()

    def __len__(self):
        with self._cv:
            return len(self._items)


@dataclass
class Command:
    """An engine command: the unique key, the batch's lengths ("bind the sequence
    length information of a batch with the command") and, for the first stage, the
    token ids [B, max_len] (host memory)."""
    key: int
    batch_id: int
    seq_lens: list
    max_len: int
    tokens: object = None

    @property
    def batch(self) -> int:
        return len(self.seq_lens)

    def rows(self, drce: bool = True) -> int:
        """Rows of the activations between stages: T with DRCE, B * max_len without."""
        return sum(self.seq_lens) if drce else self.batch * self.max_len


SHUTDOWN = -1


@dataclass
class Trace:
    """Run-level event log (time, stage, kind, key) for the ordering tests."""
    events: list = field(default_factory=list)
    lock: threading.Lock = field(default_factory=threading.Lock)

    def add(self, stage: int, kind: str, key: int) -> None:
        with self.lock:
            self.events.append((time.monotonic(), stage, kind, key))

    def keys(self, stage: int, kind: str = "run") -> list:
        with self.lock:
            return [k for _, s, kd, k in self.events if s == stage and kd == kind]


class StageFailed(RuntimeError):
    def __init__(self, key: int, stage: int, cause: BaseException):
        super().__init__(f"batch key {key} failed in stage {stage}: {cause!r}")
        self.key, self.stage, self.cause = key, stage, cause


class _Poison:
    """Travels downstream in place of the activations of a failed key (local transport)."""

    def __init__(self, err: StageFailed):
        self.err = err


class StageWorker:
    """One worker of one stage.  A dispatcher thread receives commands and hands
    each one to a pool of admit threads (the paper's per-command worker threads that "compete for the
    lock"), which insert it into the consistency queue under the engine's key; one compute thread pops
    keys in order, obtains the activations (the first stage builds them from the tokens), runs the
    stage and passes the result on.  ``admit_delay`` (tests) injects a random delay per command."""

    def __init__(self, stage: int, n_stages: int, runner, link, *, admit_threads: int = 4,
                 admit_delay: float = 0.0, trace: Trace | None = None, seed: int = 0):
        self.stage, self.n_stages, self.runner, self.link = stage, n_stages, runner, link
        self.q = ConsistencyQueue()
        self.trace = trace
        self.admit_delay = admit_delay
        self._rng = random.Random(seed * 7919 + stage)
        self._admit = ThreadPoolExecutor(max(1, admit_threads), thread_name_prefix=f"admit{stage}")
        self._threads = []
        self.transfers = 0  # activation sends from this worker
        self.error: BaseException | None = None

    @property
    def first(self) -> bool:
        return self.stage == 0

    @property
    def last(self) -> bool:
        return self.stage == self.n_stages - 1

    def start(self) -> "StageWorker":
        for fn, name in ((self._dispatch_loop, "dispatch"), (self._compute_loop, "compute")):
            t = threading.Thread(target=fn, name=f"stage{self.stage}-{name}", daemon=True)
            t.start()
            self._threads.append(t)
        return self

    def join(self, timeout: float | None = None) -> None:
        for t in self._threads:
            t.join(timeout)
        self._admit.shutdown(wait=True)

    def _admit_one(self, cmd: Command) -> None:
        if self.admit_delay:
            time.sleep(self._rng.random() * self.admit_delay)
        if self.trace:
            self.trace.add(self.stage, "admit", cmd.key)
        self.q.insert(cmd.key, cmd)

    def _dispatch_loop(self) -> None:
        pending = []
        try:
            while True:
                cmd = self.link.recv_command(self.stage)
                if cmd is None or cmd.key == SHUTDOWN:
                    break
                pending.append(self._admit.submit(self._admit_one, cmd))
            for f in pending:
                f.result()
        except BaseException as e:  # noqa: BLE001 -- surfaced through self.error
            self.error = e
        finally:
            self.q.close()

    def _compute_loop(self) -> None:
        try:
            if hasattr(self.runner, "setup"):
                self.runner.setup()
            while True:
                try:
                    key, cmd = self.q.pop_next()
                except Closed:
                    break
                x = None if self.first else self.link.recv_act(self.stage, cmd)
                if self.trace:
                    self.trace.add(self.stage, "run", key)
                if isinstance(x, _Poison):
                    out = x
                else:
                    try:
                        out = self.runner(cmd, x)
                    except Exception as e:  # noqa: BLE001 -- fail this key, keep the pipeline alive
                        out = _Poison(StageFailed(key, self.stage, e))
                if self.last:
                    self.link.deliver(self.stage, cmd, out)
                else:
                    self.link.send_act(self.stage, cmd, out)
                    self.transfers += 1
        except BaseException as e:  # noqa: BLE001
            self.error = e
            raise


class Engine:
    """The engine: ``submit`` returns a future at once; ``lanes`` dispatch
    threads (default 2 * pp, enough in-flight batches to fill the pipeline) each take the
    next unique key and broadcast the command.  The future resolves with the last stage's output."""

    def __init__(self, link, n_lanes: int, *, lane_delay: float = 0.0, seed: int = 0, trace: Trace | None = None):
        self.link = link
        self.counter = LoopCounter()
        self._lanes = ThreadPoolExecutor(max(1, n_lanes), thread_name_prefix="lane")
        self._futures: dict[int, Future] = {}
        self._cmds: dict[int, Command] = {}
        self._cv = threading.Condition()
        self._batch_ids = LoopCounter()
        self._lane_delay = lane_delay
        self._rng = random.Random(seed)
        self._rng_lock = threading.Lock()
        self._inflight = []
        self._closed = False
        self.drained = False  # every submitted batch has been dispatched (set by shutdown)
        self.trace = trace

    def submit(self, tokens, seq_lens, max_len: int | None = None) -> Future:
        """Queue one batch: tokens [B, max_len] host int32 (numpy or torch), seq_lens [B]."""
        if self._closed:
            raise RuntimeError("submit after shutdown")
        fut = Future()
        lens = [int(x) for x in seq_lens]
        S = int(max_len if max_len is not None else tokens.shape[1])
        bid = self._batch_ids.next()
        self._inflight.append(self._lanes.submit(self._launch, fut, bid, tokens, lens, S))
        return fut

    def _launch(self, fut: Future, bid: int, tokens, lens, S) -> None:
        if self._lane_delay:
            with self._rng_lock:
                d = self._rng.random() * self._lane_delay
            time.sleep(d)
        key = self.counter.next()  # "get an updated value from the loop data structure as the unique key"
        cmd = Command(key, bid, lens, S, tokens)
        with self._cv:
            self._futures[key] = fut
            self._cmds[key] = cmd
            self._cv.notify_all()
        if self.trace:
            self.trace.add(-1, "key", key)
        if self._lane_delay:
            with self._rng_lock:
                d = self._rng.random() * self._lane_delay
            time.sleep(d)
        self.link.broadcast_command(cmd)

    def command(self, key: int, timeout: float | None = None) -> Command:
        """The command registered under `key` (blocks until a lane took that key)."""
        with self._cv:
            if not self._cv.wait_for(lambda: key in self._cmds, timeout):
                raise TimeoutError(f"no command with key {key}")
            return self._cmds[key]

    def complete(self, key: int, out) -> None:
        with self._cv:
            fut = self._futures.pop(key)
            self._cmds.pop(key, None)
        if isinstance(out, _Poison):
            fut.set_exception(out.err)
        else:
            fut.set_result(out)

    def shutdown(self) -> None:
        """Finish dispatching every submitted batch, then tell every worker to stop."""
        self._closed = True
        for f in self._inflight:
            f.result()
        self._lanes.shutdown(wait=True)
        self.drained = True
        self.link.broadcast_command(Command(SHUTDOWN, -1, [], 0))


# ----------------------------------------------------------------------------- in-process transport
class LocalLink:
    """All stages are threads of this process.  Activations are handed over through one FIFO per link
    (keys arrive in order by construction; the key is checked); on the GPU the producer records a CUDA
    event on its stream and the consumer's stream waits on it."""

    def __init__(self, n_stages: int):
        self.n = n_stages
        self.inbox = [queue.Queue() for _ in range(n_stages)]
        self.links = [queue.Queue() for _ in range(max(n_stages - 1, 0))]
        self.engine: Engine | None = None

    def broadcast_command(self, cmd: Command) -> None:
        for s in range(self.n):
            self.inbox[s].put(cmd)

    def recv_command(self, stage: int) -> Command:
        return self.inbox[stage].get()

    def send_act(self, stage: int, cmd: Command, x) -> None:
        ev = None
        if not isinstance(x, _Poison) and getattr(x, "is_cuda", False):
            import torch
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
        self.links[stage].put((cmd.key, x, ev))

    def recv_act(self, stage: int, cmd: Command):
        key, x, ev = self.links[stage - 1].get()
        if key != cmd.key:
            raise ProtocolError(f"stage {stage} expected key {cmd.key}, received {key}")
        if ev is not None:
            import torch
            cur = torch.cuda.current_stream()
            cur.wait_event(ev)
            x.record_stream(cur)
        return x

    def deliver(self, stage: int, cmd: Command, out) -> None:
        if not isinstance(out, _Poison) and getattr(out, "is_cuda", False):
            import torch
            torch.cuda.current_stream().synchronize()  # the future's value is complete when it resolves
        self.engine.complete(cmd.key, out)


class LocalPipeline:
    """A pp-stage NBPP pipeline inside one process: ``runners[i](cmd, x) -> y`` runs stage i
    (``EnergonStageRunner`` on the GPU).  ``submit`` / ``shutdown`` as ``Engine``."""

    def __init__(self, runners, *, n_lanes: int | None = None, admit_threads: int = 4,
                 admit_delay: float = 0.0, lane_delay: float = 0.0, seed: int = 0, trace: Trace | None = None):
        n = len(runners)
        self.trace = trace
        self.link = LocalLink(n)
        self.engine = Engine(self.link, n_lanes or 2 * n, lane_delay=lane_delay, seed=seed, trace=trace)
        self.link.engine = self.engine
        self.workers = [StageWorker(i, n, r, self.link, admit_threads=admit_threads,
                                    admit_delay=admit_delay, trace=trace, seed=seed).start()
                        for i, r in enumerate(runners)]

    def submit(self, tokens, seq_lens, max_len: int | None = None) -> Future:
        return self.engine.submit(tokens, seq_lens, max_len)

    def shutdown(self, timeout: float | None = 60.0) -> None:
        self.engine.shutdown()
        for w in self.workers:
            w.join(timeout)
        errs = [w.error for w in self.workers if w.error is not None]
        if errs:
            raise errs[0]

    @property
    def transfers(self) -> int:
        return sum(w.transfers for w in self.workers)


# ----------------------------------------------------------------------------- torch.distributed transport
class DistLink:
    """One process per (stage, TP rank), rank = stage * tp + tp_rank, the engine on rank 0.

    * commands: rank 0 -> every rank over ``cmd_group`` (gloo), as [header int64 (key, batch_id, B, S,
      has_tokens, lens...)] + [tokens int32 [B, S]] (tokens to the first stage only);
    * activations: stage s, TP rank r -> stage s+1, TP rank r, ``dist.send`` / ``dist.recv`` of the
      [rows, H] fp32 residual rows on ``act_group`` (NCCL over NVLink on the GPU box; gloo in the CPU
      tests) -- exactly pp - 1 transfers per batch per TP rank, matched by the key order alone;
    * results: the last stage's TP rank 0 -> rank 0 over ``res_group``, received in key order by the
      engine's result thread.
    ``act_shape(cmd)`` / ``out_shape(cmd)`` give the receive buffers (shape, dtype, device)."""

    HDR = 8  # fixed preamble: [n_header_words, n_token_words]

    def __init__(self, pp: int, tp: int, act_spec, out_spec, *, cmd_group=None, act_group=None, res_group=None,
                 stage_via_host: bool = False):
        """stage_via_host: move CUDA activations through host memory (for a gloo `act_group`,
        e.g. several stages sharing one GPU in a test; NCCL sends device memory directly)."""
        import torch.distributed as dist
        self.dist = dist
        self.pp, self.tp = pp, tp
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        if self.world != pp * tp:
            raise ValueError(f"world size {self.world} != pp * tp = {pp * tp}")
        self.stage, self.tp_rank = divmod(self.rank, tp)
        self.act_spec, self.out_spec = act_spec, out_spec
        self.cmd_group = cmd_group
        self.act_group = act_group
        self.res_group = res_group
        self.engine: Engine | None = None
        self._local_inbox: queue.Queue = queue.Queue()
        self._send_lock = threading.Lock()
        self._res_thread = None
        self.result_src = (pp - 1) * tp
        self.via_host = stage_via_host

    # -- engine side (rank 0)
    def broadcast_command(self, cmd: Command) -> None:
        import numpy as np
        import torch
        with self._send_lock:  # one sender at a time on the gloo command group
            for r in range(self.world):
                stage = r // self.tp
                with_tokens = cmd.key != SHUTDOWN and stage == 0
                if r == self.rank:
                    self._local_inbox.put(cmd)
                    continue
                hdr = torch.tensor([cmd.key, cmd.batch_id, cmd.batch, cmd.max_len, int(with_tokens)] + list(cmd.seq_lens),
                                   dtype=torch.int64)
                tok = None
                if with_tokens:
                    tok = torch.as_tensor(np.ascontiguousarray(np.asarray(cmd.tokens, dtype=np.int32)))
                pre = torch.zeros(self.HDR, dtype=torch.int64)
                pre[0], pre[1] = hdr.numel(), 0 if tok is None else tok.numel()
                self.dist.send(pre, r, group=self.cmd_group)
                self.dist.send(hdr, r, group=self.cmd_group)
                if tok is not None:
                    self.dist.send(tok.reshape(-1), r, group=self.cmd_group)

    def start_results(self) -> None:
        """Rank 0: receive the last stage's outputs in key order (when the last stage is remote)."""
        if self.rank != 0 or self.result_src == 0:
            return

        def loop():
            key = 0
            while True:
                try:
                    cmd = self.engine.command(key, timeout=0.5)
                except TimeoutError:
                    if self.engine.drained and not self.engine._futures:
                        return
                    continue
                shape, dtype, device = self.out_spec(cmd)
                import torch
                out = torch.empty(shape, dtype=dtype, device="cpu" if self.via_host else device)
                self.dist.recv(out, self.result_src, group=self.res_group)
                self.engine.complete(key, out)
                key += 1

        self._res_thread = threading.Thread(target=loop, name="results", daemon=True)
        self._res_thread.start()

    def join_results(self, timeout: float | None = None) -> None:
        if self._res_thread is not None:
            self._res_thread.join(timeout)

    # -- worker side
    def recv_command(self, stage: int) -> Command:
        import torch
        if self.rank == 0:
            return self._local_inbox.get()
        pre = torch.zeros(self.HDR, dtype=torch.int64)
        self.dist.recv(pre, 0, group=self.cmd_group)
        hdr = torch.zeros(int(pre[0]), dtype=torch.int64)
        self.dist.recv(hdr, 0, group=self.cmd_group)
        h = hdr.tolist()
        key, bid, B, S, has_tok = h[:5]
        tok = None
        if has_tok:
            t = torch.zeros(int(pre[1]), dtype=torch.int32)
            self.dist.recv(t, 0, group=self.cmd_group)
            tok = t.reshape(B, S).numpy()
        return Command(key, bid, h[5:5 + B], S, tok)

    def _host(self, x):
        if self.via_host and getattr(x, "is_cuda", False):
            return x.to("cpu")  # synchronous copy: the stream's work on x is complete
        return x.contiguous()

    def send_act(self, stage: int, cmd: Command, x) -> None:
        if isinstance(x, _Poison):
            raise x.err
        self.dist.send(self._host(x), self.rank + self.tp, group=self.act_group)

    def recv_act(self, stage: int, cmd: Command):
        import torch
        shape, dtype, device = self.act_spec(cmd)
        if self.via_host and str(device).startswith("cuda"):
            h = torch.empty(shape, dtype=dtype)
            self.dist.recv(h, self.rank - self.tp, group=self.act_group)
            return h.to(device)
        x = torch.empty(shape, dtype=dtype, device=device)
        self.dist.recv(x, self.rank - self.tp, group=self.act_group)
        return x

    def deliver(self, stage: int, cmd: Command, out) -> None:
        if self.tp_rank != 0:
            return  # every TP rank holds the replicated result; rank 0 of the stage reports it
        if self.rank == 0:
            if not isinstance(out, _Poison) and getattr(out, "is_cuda", False):
                import torch
                torch.cuda.current_stream().synchronize()
            self.engine.complete(cmd.key, out)
            return
        if isinstance(out, _Poison):
            raise out.err
        self.dist.send(self._host(out), 0, group=self.res_group)


# ----------------------------------------------------------------------------- the GPU stage runner
class EnergonStageRunner:
    """Stage i of a plan: layers [l0, l1) of one context (or a local TP group) through
    ``energon_forward_stage``.  The first stage copies the command's host tokens to the device; the
    last returns the final [B, S, H] output (cfg dtype), the others the fp32 [rows, H] residual rows.
    Runs on the compute thread's current CUDA stream (``setup`` gives the thread its own stream)."""

    def __init__(self, ctxs, layer_begin: int, layer_end: int, *, first: bool, last: bool, hidden: int,
                 out_dtype, device: int = 0, drce: bool = True, own_stream: bool = True):
        self.ctxs = ctxs if isinstance(ctxs, (list, tuple)) else [ctxs]
        self.l0, self.l1, self.first, self.last = layer_begin, layer_end, first, last
        self.H, self.out_dtype, self.device, self.drce = hidden, out_dtype, device, drce
        self.own_stream = own_stream

    def setup(self) -> None:
        import torch
        torch.cuda.set_device(self.device)
        if self.own_stream:
            torch.cuda.set_stream(torch.cuda.Stream(self.device))

    def __call__(self, cmd: Command, x):
        import numpy as np
        import torch

        from . import energon
        st = torch.cuda.current_stream()
        B, S = cmd.batch, cmd.max_len
        tok = None
        if self.first:
            host = torch.from_numpy(np.ascontiguousarray(np.asarray(cmd.tokens, dtype=np.int32))).pin_memory()
            tok = host.to(f"cuda:{self.device}", non_blocking=True)
        if self.last:
            out = torch.empty((B, S, self.H), dtype=self.out_dtype, device=f"cuda:{self.device}")
            kind = energon.STAGE_FINAL
        else:
            out = torch.empty((cmd.rows(self.drce), self.H), dtype=torch.float32, device=f"cuda:{self.device}")
            kind = energon.STAGE_PACKED
        if len(self.ctxs) == 1:
            energon.energon_forward_stage(self.ctxs[0], cmd.seq_lens, S, self.l0, self.l1, kind, out, tokens=tok, x=x,
                                          stream=st)
        else:
            energon.energon_forward_stage_group(self.ctxs, cmd.seq_lens, S, self.l0, self.l1, kind, out, tokens=tok,
                                                x=x, stream=st)
        return out
