"""The slice-sharded multi-rank frame on the GPU: world sizes 2 and 4 (a depth-1 / -2
subtree per rank: the ranks slice only the top levels of the whole G-buffer, then their own
subtree) and 3 (slice index ranges), on the interior, Cornell and mesh scenes, every rank on GPU 0 with the gloo transport (one GPU is available to the
tests; the production path gathers with NCCL inside lmc_resolve_image, one rank per GPU).  Each
rank runs the CUDA path on its share (lmc_get_partition), packs its rows (lmc_resolve_rows), the
tiles are gathered to rank 0 and scattered (lmc_scatter_rows): the image must equal the
single-rank image bit for bit, and each rank's slicing must equal the single-rank slicing on its
rows, since a slice's computation does not depend on which rank runs it."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import scenegen  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q, partition=0):
    import torch.distributed as dist

    from paper_2202_12567_b200 import dist as pdist
    from paper_2202_12567_b200 import lmc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    x = scenegen.make_inputs(name)
    fr = lmc.Frame(x, rank=rank, world=world, partition=partition)
    fr.build_slices()
    sf, rf = fr.partition()
    counts = pdist.row_counts(rf)
    st = fr.stats()
    assert st["rows"] == counts[rank] and st["slice_begin"] == sf[rank] and st["slice_end"] == sf[rank + 1]
    off, rows = fr.slices()
    fr.sample_pass1()
    fr.coarsen_cut()
    fr.sample_pass2()
    fr.complete()
    tile = torch.zeros(counts[rank] * 4, device="cuda")
    fr.resolve_rows(tile)
    allrows = pdist.gather_rows(tile, counts)
    if partition == 1:   # interleaved: every rank slices the whole frame
        q.put(("rows", rank, 0, rows.size, rows.copy()))
    else:
        q.put(("rows", rank, int(rf[rank]), int(rf[rank + 1]), rows[rf[rank]:rf[rank + 1]].copy()))
    if rank == 0:
        img = torch.zeros(x.height * x.width * 3, device="cuda")
        fr.scatter_rows(allrows, img)
        torch.cuda.synchronize()
        q.put(("img", img.cpu().numpy()))
    dist.barrier()
    fr.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,partition", [("t_interior", 2, 0), ("t_interior", 3, 0), ("t_interior", 4, 0),
                                                  ("c1", 4, 0), ("t_mesh", 2, 0), ("t_interior", 2, 1),
                                                  ("t_interior", 3, 1), ("c1", 4, 1), ("t_cornell", 5, 1)])
def test_sharded_frame_equals_single_rank(name, world, partition):
    """partition 0: slicing subtrees (P = 2^k) or slice ranges; 1: interleaved slices (the draws
    keyed by the global slice id, so the image is bit-identical either way)"""
    from paper_2202_12567_b200 import lmc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, partition)) for r in range(world)]
    for p in procs:
        p.start()
    items = [q.get(timeout=600) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = [it[1] for it in items if it[0] == "img"][0]
    parts = [it for it in items if it[0] == "rows"]
    x = scenegen.make_inputs(name)
    fr = lmc.Frame(x)
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    ref = img.cpu().numpy()
    _, rows1 = fr.slices()
    fr.close()
    for _, r, a, b, rws in parts:   # each rank's slicing equals the single-rank slicing on its rows
        assert np.array_equal(rws, rows1[a:b]), f"rank {r}: slicing differs"
    assert np.array_equal(got, ref)
    assert np.count_nonzero(ref) > 0.5 * ref.size
