"""World-size-2 gloo test of the slice-sharded gather on CPU: each rank takes its
slice range, produces its packed tile (here from the oracle's per-slice rows, standing in for
lmc_resolve_rows), and the gathered slice-ordered rows equal the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import scenegen
from paper_2202_12567_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = scenegen.make_inputs(name)
    o = oracle.Oracle(x)
    off, rows = o.slices()
    S = off.size - 1
    s0, s1 = pdist.slice_range(S, rank, world)
    res = o.run_slices(list(range(s0, s1)), stage=4)
    tile = torch.from_numpy(np.concatenate([r["rgb"] for r in res]).astype(np.float32)) if res else torch.zeros(0, 3)
    counts = pdist.row_counts(off, world)
    assert counts[rank] == tile.shape[0]
    allrows = pdist.gather_rows(tile, counts)
    if rank == 0:
        q.put(allrows.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_equals_single_process(world):
    name = "t_cornell"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = scenegen.make_inputs(name)
    o = oracle.Oracle(x)
    off, rows = o.slices()
    ref = np.concatenate([r["rgb"] for r in o.run_slices(list(range(off.size - 1)), stage=4)]).astype(np.float32)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
    # scatter into the image by the slice-ordered rows (what lmc_scatter_rows does on the GPU)
    img = np.zeros((x.width * x.height, 3), np.float32)
    img[x.gbuf["pixel"][rows]] = got
    assert np.count_nonzero(img.any(1)) > 0.9 * x.m


def test_row_counts_cover_every_row():
    for S, world in [(16, 2), (16, 3), (2048, 8), (7, 4)]:
        off = np.cumsum([0] + [10 + (s % 3) for s in range(S)])
        c = pdist.row_counts(off, world)
        assert sum(c) == off[-1]
        ranges = [pdist.slice_range(S, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == S
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
