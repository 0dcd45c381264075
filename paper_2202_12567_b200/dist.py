"""Multi-GPU plumbing for the slice-sharded frame.

Slices are independent after slicing.  With P = 2^k ranks, rank r owns the
r-th depth-k subtree of the slicing (every rank slices the top k levels of the whole G-buffer,
then only inside its subtree); other P split the slice index range; with lmc_config.partition = 1
(the bench's default at N > 1) rank r takes slices r, r + P, ... of a full slicing, which balances
the ranks' completion work.  The library reports the
shares (Frame.partition()).  The production image assembly is inside the library: the ranks pass
an NCCL id (lmc_nccl_unique_id on rank 0, broadcast with torch.distributed) and
lmc_resolve_image gathers every rank's packed rows to rank 0 over NVLink (one NCCL group of
send / receive pairs).  This module is the alternative transport through torch.distributed (gloo
in the CPU tests and the single-GPU multi-rank test): each rank packs its rows (lmc_resolve_rows,
4 floats per row: r, g, b, pixel index), rank 0 gathers them and scatters (lmc_scatter_rows).
"""
from __future__ import annotations


def row_counts(row_first):
    """rows per rank from the partition's row offsets (world + 1 entries, identical on every rank)"""
    return [int(row_first[r + 1]) - int(row_first[r]) for r in range(len(row_first) - 1)]


def gather_rows(tile, counts, group=None, dst=0):
    """Gather the per-rank packed tiles (rows x 4 floats) to rank `dst` (padded to the largest tile
    so that one equal-size collective moves them); returns the concatenation (sum(counts) x 4) on
    `dst` and None elsewhere."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    rank = dist.get_rank(group)
    mx = max(counts)
    pad = torch.zeros(mx * 4, dtype=tile.dtype, device=tile.device)
    pad[: counts[rank] * 4] = tile.reshape(-1)[: counts[rank] * 4]
    dev = pad.device
    if pad.is_cuda and dist.get_backend(group) == "gloo":   # gloo moves host tensors
        pad = pad.cpu()
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][: counts[r] * 4] for r in range(world)]).view(-1, 4).to(dev)
