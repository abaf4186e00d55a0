"""Multi-process (world_size 2, gloo, CPU) tests of the sharding and statistics reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_17770_b200 import dist as cdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_stats(rank: int) -> dict:
    g = torch.Generator().manual_seed(100 + rank)
    st = {k: int(torch.randint(0, 10**9, (1,), generator=g)) for k in cdist.SUM_KEYS}
    st.update({k: int(torch.randint(0, 128, (1,), generator=g)) for k in cdist.MAX_KEYS})
    st["unique_hist"] = torch.randint(0, 1000, (129,), generator=g).tolist()
    st["sum_sq_err"] = float(torch.rand(1, generator=g, dtype=torch.float64)) * 1e-3
    st["max_abs_err"] = float(torch.rand(1, generator=g, dtype=torch.float64))
    return st


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        red = cdist.reduce_stats(_fake_stats(rank))
        mx = cdist.max_over_ranks(float(rank) + 0.5)
        q.put((rank, red, mx))
    finally:
        dist.destroy_process_group()


def test_reduce_stats_world2_matches_rank_ordered_sum():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = cdist.reduce_stats_local([_fake_stats(r) for r in range(world)])
    for rank, red, mx in res:
        assert red == expect          # bitwise, on every rank (fp64 sums in rank order)
        assert mx == world - 0.5


def test_frame_shards_partition_the_batch():
    for total in (64, 65, 7):
        for world in (1, 2, 4, 8):
            frames = [f for r in range(world) for f in cdist.frame_shard(total, world, r)]
            assert frames == list(range(total))


def test_weak_frames_distinct_rng_indices():
    idx = [cdist.weak_frames(64, r)[1] + f for r in range(8) for f in range(64)]
    assert len(set(idx)) == 8 * 64
    assert cdist.weak_frames(64, 1)[0][0] == 0   # path position wraps every 64 frames


def test_single_process_reduce_is_identity():
    st = _fake_stats(0)
    red = cdist.reduce_stats(st)
    assert red["texel_evals"] == st["texel_evals"] and red["unique_hist"] == st["unique_hist"]
