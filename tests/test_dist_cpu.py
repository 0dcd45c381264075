"""World-size 2 / 3 gloo tests of the multi-rank frame's host logic on CPU (DESIGN.md §8,
SURVEY §8(e)): the ranks' shares planned by the library (lmc_plan_partition, no GPU needed), the
packed-row gather to rank 0 and the scatter into the image.  The per-slice rows come from the
oracle, standing in for lmc_resolve_rows; the gathered image must equal the single-process one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import scenegen
from paper_2202_12567_b200 import dist as pdist
from paper_2202_12567_b200 import lmc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(x, rows, rgb):
    """(r, g, b, pixel index bits) float32 rows, as lmc_resolve_rows writes them"""
    t = np.zeros((rows.size, 4), np.float32)
    t[:, :3] = rgb
    t[:, 3] = x.gbuf["pixel"][rows].astype(np.int32).view(np.float32)
    return t


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = scenegen.make_inputs(name)
    o = oracle.Oracle(x)
    sf, rf, S = lmc.plan_partition(x.m, x.cfg.slice_target, world)
    res = o.run_slices(list(range(sf[rank], sf[rank + 1])), stage=4)
    tile = np.concatenate([_pack(x, r["rows"], r["rgb"]) for r in res]) if res else np.zeros((0, 4), np.float32)
    counts = pdist.row_counts(rf)
    assert counts[rank] == tile.shape[0]
    allrows = pdist.gather_rows(torch.from_numpy(tile), counts)
    if rank == 0:
        q.put(allrows.numpy())
    else:
        assert allrows is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_to_root_equals_single_process(world):
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
    ref = np.concatenate([_pack(x, r["rows"], r["rgb"]) for r in o.run_slices(list(range(off.size - 1)), stage=4)])
    assert np.array_equal(got, ref)                     # rank order = slice order
    img = np.zeros((x.width * x.height, 3), np.float32)  # what lmc_scatter_rows does on the GPU
    img[got[:, 3].view(np.int32)] = got[:, :3]
    assert np.count_nonzero(img.any(1)) > 0.9 * x.m


@pytest.mark.parametrize("M,target", [(2073600, 1024), (1048576, 800), (262144, 512), (1480, 185), (12345, 100)])
def test_partition_plan(M, target):
    _, rf1, S = lmc.plan_partition(M, target, 1)
    # slice offsets of the single-rank slicing (the left child takes ceil(n / 2))
    def sizes(n):
        return [n] if n <= target else sizes((n + 1) // 2) + sizes(n - (n + 1) // 2)
    off = np.concatenate([[0], np.cumsum(sizes(M))])
    assert S == off.size - 1 and rf1.tolist() == [0, M]
    for world in (2, 3, 4, 8, 5):
        sf, rf, S2 = lmc.plan_partition(M, target, world)
        assert S2 == S and sf[0] == 0 and sf[-1] == S and rf[0] == 0 and rf[-1] == M
        assert np.all(np.diff(sf) >= 0) and np.all(np.diff(rf) >= 0)
        assert np.array_equal(rf, off[sf])             # every share is a run of whole slices
        depth = int(np.log2(world)) if world & (world - 1) == 0 else None
        if depth is not None and M > target * (1 << (depth - 1)) * 2:
            # power-of-two world: rank r's rows are the r-th subtree of depth k (sizes split by
            # ceil / floor halves, so they differ by at most one row per level)
            c = np.diff(rf)
            assert c.max() - c.min() <= depth
        else:
            assert sf.tolist() == [(S * r) // world for r in range(world + 1)]
