"""Multi-GPU plumbing for the slice-sharded frame.

Slices are independent after slicing: rank r of P owns slices
[S*r/P, S*(r+1)/P) (lmc_config.rank/world), resolves its pixels as a packed tile in slice-row
order (lmc_resolve_rows), and the tiles are gathered with one collective; rank 0 scatters the
concatenation into the image (lmc_scatter_rows).  torch.distributed is the transport (NCCL over
NVLink on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def slice_range(S: int, rank: int, world: int):
    """slices of a rank: the same integer split as lmc_create (s0 = S*rank/world)"""
    return (S * rank) // world, (S * (rank + 1)) // world


def row_counts(slice_off, world: int):
    """rows per rank, in rank order, from the slice offsets (identical on every rank)"""
    S = len(slice_off) - 1
    out = []
    for r in range(world):
        s0, s1 = slice_range(S, r, world)
        out.append(int(slice_off[s1]) - int(slice_off[s0]))
    return out


def gather_rows(tile, counts, group=None):
    """All-gather the per-rank packed tiles (rows x 3 floats, slice-row order) into the
    slice-ordered array of all rows.  Tiles are padded to the largest rank's size so one
    equal-size collective moves them; returns a tensor of sum(counts) x 3 on every rank."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    rank = dist.get_rank(group)
    mx = max(counts)
    pad = torch.zeros(mx * 3, dtype=tile.dtype, device=tile.device)
    pad[: counts[rank] * 3] = tile.reshape(-1)[: counts[rank] * 3]
    dev = pad.device
    if pad.is_cuda and dist.get_backend(group) == "gloo":   # gloo moves host tensors (CPU tests)
        pad = pad.cpu()
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][: counts[r] * 3] for r in range(world)]).view(-1, 3).to(dev)
