"""World-size-2 CPU (gloo) tests of the multi-GPU path: the DDP shard
partition and the reporting reduction bench.py uses (no
collective on the data path, one all_reduce after timing).  Also checks
that each rank's host-side descriptors (RRC rects + flips, host C++) equal
the single-process ones for the same indices."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2404_00509_b200 import _native as N
    from paper_2404_00509_b200.ddp import rank_shard, reduce_timing
    n, seed, epoch = 1000, 7, 3
    idx = rank_shard(seed, epoch, n, rank, ws, "stride")
    gathered = [None] * ws
    dist.all_gather_object(gathered, idx.tolist())
    # host descriptors of this rank's shard (rects/flips keyed by index)
    w = np.full(n, 320, np.uint16)
    h = np.full(n, 240, np.uint16)
    s = np.zeros(len(idx), N._np_dtypes()[0])
    ii = np.ascontiguousarray(idx, np.int64)
    N.check(N.lib().essl_rrc_batch(seed, epoch, N.ptr(ii), len(ii), N.ptr(w), N.ptr(h), 0.08, 1.0,
                                   0.75, 4.0 / 3.0, N.ptr(s)), "essl_rrc_batch")
    rects = [[int(r["x"]), int(r["y"]), int(r["w"]), int(r["h"]), int(r["flip"])] for r in s]
    all_rects = [None] * ws
    dist.all_gather_object(all_rects, rects)
    # reporting reduction: max time, summed images
    red = reduce_timing([10.0 + rank, 100 * (rank + 1), 20.0 - rank, 7 * (rank + 1)])
    if rank == 0:
        q.put((gathered, all_rects, red))
    dist.barrier()
    dist.destroy_process_group()


def test_ddp_shards_and_reduction_gloo():
    sys.path.insert(0, str(ROOT))
    from paper_2404_00509_b200 import _native as N
    from paper_2404_00509_b200.rng import epoch_permutation
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    gathered, all_rects, red = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    perm = epoch_permutation(7, 3, 1000)
    # disjoint, covering, and rank r holds perm[r::2] in order
    assert sorted(gathered[0] + gathered[1]) == list(range(1000))
    for r in range(ws):
        assert gathered[r] == perm[r::ws].tolist()
    # per-rank descriptors == single-process descriptors of the same indices
    idx = np.ascontiguousarray(perm, np.int64)
    w = np.full(1000, 320, np.uint16)
    h = np.full(1000, 240, np.uint16)
    s = np.zeros(1000, N._np_dtypes()[0])
    N.check(N.lib().essl_rrc_batch(7, 3, N.ptr(idx), 1000, N.ptr(w), N.ptr(h), 0.08, 1.0, 0.75,
                                   4.0 / 3.0, N.ptr(s)), "essl_rrc_batch")
    single = {int(i): [int(r["x"]), int(r["y"]), int(r["w"]), int(r["h"]), int(r["flip"])]
              for i, r in zip(idx, s)}
    for r in range(ws):
        for i, rect in zip(gathered[r], all_rects[r]):
            assert single[i] == rect
    assert red == (11.0, 300.0, 20.0, 21.0)


def _gpu_worker(rank, ws, port, path, q):
    """One DDP rank (own process, own CUDA context on the one GPU): its shard
    of an epoch through the GPU loader, digests per dataset index, then the
    bench's reporting reduction over gloo."""
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import hashlib
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200.ddp import reduce_timing
    torch.cuda.set_device(0)
    cfg = E.LoaderConfig(data=path, batch_size=8, res=96, mask_ratio=0.75, rank=rank,
                         world_size=ws, shard_mode="stride", out_dtype="bfloat16")
    out, nb = {}, 0
    with E.Loader(cfg) as loader:
        for b in loader.epoch(4):
            nb += 1
            for s in range(len(b)):
                out[int(b.indices[s])] = (
                    hashlib.sha256(b.pixels[s].cpu().view(torch.int16).numpy().tobytes()).hexdigest(),
                    b.mask[s].cpu().tolist())
    red = reduce_timing([1.0 + rank, float(len(out)), 0.0, 0.0])
    gathered = [None] * ws
    dist.all_gather_object(gathered, out)
    if rank == 0:
        q.put((gathered, red, nb))
    dist.barrier()
    dist.destroy_process_group()


import pytest  # noqa: E402


@pytest.mark.gpu
def test_two_ranks_on_gpu_equal_single_process(tmp_path):
    """2 DDP ranks (gloo for the reporting collective, no collective on the
    data path) decode disjoint shards whose union equals the single-process
    epoch, sample for sample."""
    sys.path.insert(0, str(ROOT))
    import hashlib
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_00509_b200 as E
    path = str(tmp_path / "d.essl")
    E.build_synthetic(path, 37, 256, 95, seed=8)
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, ws, port, path, q)) for r in range(ws)]
    for p in procs:
        p.start()
    gathered, red, nb = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    union = {}
    for g in gathered:
        assert not set(g) & set(union)  # disjoint shards
        union.update(g)
    cfg = E.LoaderConfig(data=path, batch_size=8, res=96, mask_ratio=0.75, out_dtype="bfloat16")
    single = {}
    with E.Loader(cfg) as loader:
        for b in loader.epoch(4):
            for s in range(len(b)):
                single[int(b.indices[s])] = (
                    hashlib.sha256(b.pixels[s].cpu().view(torch.int16).numpy().tobytes()).hexdigest(),
                    b.mask[s].cpu().tolist())
    assert union == single
    assert red == (2.0, 37.0, 0.0, 0.0)
