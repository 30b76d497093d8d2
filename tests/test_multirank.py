"""World-size-2 gloo run of the multi-GPU host logic (CPU only)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2212_01185_b200.shard import aggregate_msubpx, shard_range, weak_seeds


def test_shard_range_partitions():
    for n in (1, 7, 24, 256):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                lo, hi = shard_range(n, r, world)
                cover.extend(range(lo, hi))
                assert (hi - lo) in (n // world, n // world + 1)
            assert cover == list(range(n))
    assert list(weak_seeds(24, 1)) == list(range(24, 48))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2212_01185_b200.shard import max_over_ranks
    t = max_over_ranks(1.5 + rank)            # rank 1 is the slow one
    lo, hi = shard_range(256, rank, world)
    q.put((rank, t, lo, hi))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_max_and_shards():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2.5, 2.5]
    assert (res[0][2], res[0][3], res[1][2], res[1][3]) == (0, 128, 128, 256)
    assert aggregate_msubpx(3e6, 2, 2.5) == pytest.approx(2.4)
