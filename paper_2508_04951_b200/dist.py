"""Pulse sharding across ranks (one process per GPU) -- no collective on the data path.

Pulses are independent ("process receive signals on a pulse-to-pulse basis"), so a
pulse train of P pulses is split into contiguous blocks: rank r of G owns
[r*P//G, (r+1)*P//G).  torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only
after the timed region: the max-over-ranks elapsed time and, optionally, gathering results.
"""
from __future__ import annotations


def shard_range(pulses: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of the pulse train owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    if pulses < 0:
        raise ValueError("pulses must be >= 0")
    return rank * pulses // world, (rank + 1) * pulses // world


def max_over_ranks(value: float, device=None) -> float:
    """max of a per-rank scalar (e.g. elapsed ms) over the default process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_pulses(y_local, pulses: int, device=None):
    """All-gather each rank's output block [lo, hi) into the full [pulses, n] train (off the hot path)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return y_local
    world = dist.get_world_size()
    sizes = [shard_range(pulses, r, world) for r in range(world)]
    maxb = max(hi - lo for lo, hi in sizes)
    n = y_local.shape[-1]
    buf = torch.zeros((maxb, n), dtype=y_local.dtype, device=y_local.device)
    buf[: y_local.shape[0]] = y_local
    # gloo/nccl all_gather on real views (complex tensors viewed as float)
    parts = [torch.zeros_like(torch.view_as_real(buf)) for _ in range(world)]
    dist.all_gather(parts, torch.view_as_real(buf).contiguous())
    out = [torch.view_as_complex(p)[: hi - lo] for p, (lo, hi) in zip(parts, sizes)]
    return torch.cat(out, dim=0)
