"""(batch, head) sharding of the ASA forward over the GPUs of one box.

Each (b, h) unit's mask and attention depend only on that unit's Q, K, V
(PAPER.md P:142-154), so the path shards with no exchange step: rank r owns
a contiguous range of flattened units u = b*H + h, i.e. a contiguous slice
of [B*H, N, d], and passes the range start as ``unit_offset`` so the sampler
(keyed by the global unit index, R-1) gives the same masks as a
single-GPU run.  The only collectives are the final gather of O / LSE and the
max-over-ranks timing reduction.  Host-side plumbing only (torch.distributed
for process groups); no arithmetic of the method lives here.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def unit_range(world: int, rank: int, units: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of ``units`` for ``rank`` (floor split)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return (rank * units) // world, ((rank + 1) * units) // world


def gather_units(local: torch.Tensor, units: int, group=None, dst: int = 0):
    """Gather every rank's unit slice (leading dim) into one [units, ...]
    tensor on rank ``dst`` (None elsewhere).  Shares may be uneven."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = unit_range(world, rank, units)
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank}: expected {hi - lo} units, got {local.shape[0]}")
    biggest = max(unit_range(world, r, units)[1] - unit_range(world, r, units)[0]
                  for r in range(world))
    # gloo has no CUDA gather: stage through host memory (testing on one GPU)
    dev = local.device
    if dist.get_backend(group) == "gloo" and local.is_cuda:
        dev = torch.device("cpu")
    if hi - lo == biggest and local.device == dev and local.is_contiguous():
        pad = local  # even share: no staging copy
    else:
        pad = torch.zeros((biggest,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
        pad[:hi - lo] = local
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, parts, dst=dst, group=group)
    if rank != dst:
        return None
    out = []
    for r in range(world):
        a, b = unit_range(world, r, units)
        out.append(parts[r][:b - a])
    return torch.cat(out, 0)


def max_over_ranks(values, device=None, group=None) -> list[float]:
    """Element-wise max of a list of floats over all ranks (for timings)."""
    t = torch.tensor(list(values), dtype=torch.float64, device=_red_dev(device, group))
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


def sum_over_ranks(values, device=None, group=None) -> list[float]:
    t = torch.tensor(list(values), dtype=torch.float64, device=_red_dev(device, group))
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.tolist()


def _red_dev(device, group):
    """Reductions run where the backend can: gloo on the host."""
    if dist.is_initialized() and dist.get_backend(group) == "gloo":
        return torch.device("cpu")
    return device
