"""World-size-2 gloo run of the multi-GPU host logic (CPU only).

The workers call the SAME functions bench.py's ranks call: bench.make_images
(which partitions with shard.rank_units), shard.reduce_over_ranks for the
max-over-ranks time and the summed units, and shard.aggregate_rate for the
whole-job value."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2212_01185_b200.shard import aggregate_rate, rank_units, shard_range, split_for_devices


def test_shard_range_partitions():
    for n in (0, 1, 7, 24, 256):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                lo, hi = shard_range(n, r, world)
                cover.extend(range(lo, hi))
                assert (hi - lo) in (n // world, n // world + 1)
            assert cover == list(range(n))
    assert rank_units(24, 1, 8, "weak") == (24, 48)
    assert rank_units(256, 3, 8, "strong") == (96, 128)
    assert rank_units(8, 7, 8, "strong") == (7, 8)
    assert rank_units(1, 3, 8, "strong") == (1, 1)          # more GPUs than images: empty ranks
    with pytest.raises(ValueError):
        rank_units(4, 0, 1, "sideways")
    assert split_for_devices(5, [0, 1, 2]) == [(0, 0, 2), (1, 2, 4), (2, 4, 5)]
    assert split_for_devices(1, [0, 1]) == [(0, 0, 1)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2212_01185_b200 import shard
    out = {}
    for scaling in ("weak", "strong"):
        cfgd = dict(n=3, H=8, W=10, scaling=scaling, desc="tiny")
        imgs = bench.make_images(cfgd, rank, world, False)
        # a fake per-rank device time (rank 1 slower) through the bench's reduction
        (t_dec, t_enc), units_all = shard.reduce_over_ranks([1.5 + rank, 0.25 * (rank + 1)], 3.0 * 8 * 10 * len(imgs))
        out[scaling] = (imgs.shape[0], [int(v) for v in imgs.reshape(imgs.shape[0], -1).sum(1)], t_dec, t_enc,
                        units_all, shard.aggregate_rate(units_all, t_dec))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_bench_partition_and_reduction():
    from paper_2212_01185_b200 import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sums = {s: [int(synth.synth_1f(k, 8, 10).sum()) for k in range(6)] for s in ("weak",)}
    # weak: each rank its own 3 images (seeds 3r..3r+2); strong: 2 + 1 of 3
    assert res[0]["weak"][0] == 3 and res[1]["weak"][0] == 3
    assert res[0]["weak"][1] + res[1]["weak"][1] == sums["weak"]
    assert res[0]["strong"][0] == 2 and res[1]["strong"][0] == 1
    assert res[0]["strong"][1] + res[1]["strong"][1] == sums["weak"][:3]
    for s in ("weak", "strong"):
        for r in (0, 1):
            _, _, t_dec, t_enc, units_all, rate = res[r][s]
            assert (t_dec, t_enc) == (2.5, 0.5)                 # max over ranks
            n_all = 6 if s == "weak" else 3
            assert units_all == 3.0 * 80 * n_all               # summed units
            assert rate == pytest.approx(units_all / 2.5 / 1e6)
    assert aggregate_rate(3e6, 2.5) == pytest.approx(1.2)


def test_bench_relaunches_under_torchrun(tmp_path):
    """`bench.py --gpus 2` without a torchrun environment re-launches itself
    under torch.distributed.run; checked here through the command it builds
    (no GPU needed: the child is replaced by a stub)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, subprocess, os\n"
        "sys.path.insert(0, %r)\n"
        "import bench\n"
        "seen = []\n"
        "subprocess.call = lambda cmd: (seen.append(cmd), 0)[1]\n"
        "sys.argv = ['bench.py', '--gpus', '2', '--steps', '1']\n"
        "try:\n"
        "    bench.main()\n"
        "except SystemExit as e:\n"
        "    assert e.code == 0\n"
        "print(' '.join(seen[0]))\n"
    ) % root
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    cmd = r.stdout.strip().splitlines()[-1]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=2" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd.endswith("--gpus 2 --steps 1")
