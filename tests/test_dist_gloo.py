"""World-size-2 gloo tests of the multi-GPU host logic (GOP replicas,
BASELINE config 4): GOP sharding is a partition, the timing reduction is a max
over ranks, and the barrier/reduce plumbing bench.py uses works across
processes. CPU only (no GPU, no NCCL)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2605_20977_b200 import dist as pdist


def test_gops_partition():
    for n in (1, 7, 64):
        for world in (1, 2, 4, 8):
            seen = sorted(g for r in range(world) for g in pdist.gops_for_rank(n, r, world))
            assert seen == list(range(n))
            counts = [len(pdist.gops_for_rank(n, r, world)) for r in range(world)]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        pdist.gops_for_rank(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    d = pdist.init("gloo")
    info = pdist.rank_info()
    pdist.barrier(d)
    ms = 10.0 + 5.0 * info.rank  # per-rank "timed region"
    worst = pdist.max_over_ranks(ms, d)
    gops = pdist.gops_for_rank(64, info.rank, info.world)
    # config 4 accounting: frames of this rank's GOPs (32 each), summed
    total = pdist.sum_over_ranks(32.0 * len(gops), d)
    q.put((info.rank, worst, gops, total))
    pdist.barrier(d)
    d.destroy_process_group()


def test_two_rank_gloo_max_and_shards():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [15.0, 15.0]  # every rank reports the slowest
    assert [r[3] for r in res] == [64 * 32.0, 64 * 32.0]  # job-wide frame count
    assert sorted(res[0][2] + res[1][2]) == list(range(64))
    assert not set(res[0][2]) & set(res[1][2])


def _band_link_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    from paper_2605_20977_b200 import dist as pdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class FakeBand:  # stands in for a GPU band handle: the host logic only
        def band_export(self):
            return f"blob{rank}".encode()

        def band_link(self, up, down):
            q.put((rank, up, down))

    pdist.link_band(FakeBand(), dist)
    dist.destroy_process_group()


def test_band_link_exchanges_neighbour_blobs():
    """world-size-3 gloo: every rank is linked to exactly its row-band
    neighbours' export blobs (None at the frame edges)."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_band_link_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    got = dict((r, (u, d)) for r, u, d in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert got[0] == (None, b"blob1")
    assert got[1] == (b"blob0", b"blob2")
    assert got[2] == (b"blob1", None)
