"""Process-group plumbing for one TP group of one process per GPU (torch.distributed): the
engine-command analog of PAPER.md:368-370 -- rank 0 creates the NCCL unique id and it is broadcast;
seq_lens are SPMD arguments.  Used by bench.py; the same helpers run under gloo in the CPU tests."""
from __future__ import annotations

import os


def env_ranks():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: bytes | None, nbytes: int, src: int = 0, device=None) -> bytes:
    """Broadcast `nbytes` bytes from `src` to every rank of the default group."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device or "cpu")
    if dist.get_rank() == src:
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())


def broadcast_lengths(lens, src: int = 0, device=None) -> list:
    """The engine command's seq_lens: rank `src`'s list on every rank."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([len(lens) if dist.get_rank() == src else 0], dtype=torch.int64, device=device or "cpu")
    dist.broadcast(n, src)
    t = torch.zeros(int(n.item()), dtype=torch.int32, device=device or "cpu")
    if dist.get_rank() == src:
        t.copy_(torch.tensor(lens, dtype=torch.int32))
    dist.broadcast(t, src)
    return [int(x) for x in t.cpu().tolist()]


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
