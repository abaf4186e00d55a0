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


# ------------------------------------------------------------------------------------------
# SURVEY §8(e) on real statistics: per-frame stats of small camera-path frames, computed by the
# CPU oracle (test infrastructure), sharded over gloo ranks by frame blocks and by wave-row
# strips, reduced with reduce_frame_stats — compared with the 1-rank result.
_NF, _WF, _HF, _T = 6, 64, 42, 128      # 42 rows: 11 wave-rows, the last one ragged


def _scene(f):
    import synthetic
    return synthetic.camera_path_frame(f, _WF, _HF, _T, _T, nframes=_NF)


def _frame_records(split: str, world: int, rank: int) -> list[dict]:
    import numpy as np
    import oracle
    import synthetic
    tex = {"format": 1, "width": _T, "height": _T, "bc1": synthetic.bc1_texture(_T, _T, 3, "image")}
    nwx = (_WF + 7) // 8
    recs = []
    frames = list(cdist.frame_shard(_NF, world, rank)) if split == "frames" else list(range(_NF))
    row0, rows = (0, _HF) if split == "frames" else cdist.strip_shard(_HF, world, rank)
    if rows == 0:
        return recs
    wy0, wy1 = row0 // 4, (row0 + rows + 3) // 4
    waves = np.array([wy * nwx + wx for wy in range(wy0, wy1) for wx in range(nwx)], np.int32)
    for f in frames:
        uv, g = _scene(f)
        r = oracle.filter_waves(tex, uv, g, waves, 3, 3, seed=7, frame_index=f)
        ref = oracle.filter_waves(tex, uv, g, waves, 0, 0, seed=7, frame_index=f)
        st = oracle.frame_stats(r["rec"][wy0:wy1], r["out"][row0:row0 + rows], ref["out"][row0:row0 + rows])
        st["frame"], st["row0"] = f, row0
        recs.append(st)
    return recs


def _stats_worker(rank, world, port, split, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        red = cdist.reduce_frame_stats(_frame_records(split, world, rank))
        q.put((rank, red))
    finally:
        dist.destroy_process_group()


def _run_world(world, split):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_stats_worker, args=(r, world, port, split, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [red for _, red in sorted(res, key=lambda t: t[0])]


def _norm(st):
    return {k: ([int(x) for x in v] if k == "unique_hist" else v) for k, v in st.items()}


@pytest.mark.parametrize("world", [2, 4])
def test_frame_sharding_real_stats_bitwise_equal_to_one_rank(world):
    """Frame blocks over `world` ranks: every rank's reduced totals — integers AND the fp64 error
    sums — equal the single-rank reduction bit for bit (records reduced in frame order)."""
    one = _norm(cdist.reduce_frame_stats(_frame_records("frames", 1, 0)))
    assert one["waves_fallback"] > 0 and one["waves_exact"] > 0 and one["sum_sq_err"] > 0
    for red in _run_world(world, "frames"):
        assert _norm(red) == one


@pytest.mark.parametrize("world", [2, 4])
def test_strip_sharding_real_stats_equal_to_one_rank(world):
    """Wave-row strips over `world` ranks (4-row aligned; the 11 wave-rows split unevenly, the
    ragged last row in the last strip): integer totals bitwise equal to one rank, fp64 error
    sums equal up to the summation order of the strips."""
    one = _norm(cdist.reduce_frame_stats(_frame_records("frames", 1, 0)))
    for red in _run_world(world, "strip"):
        red = _norm(red)
        for k in cdist.SUM_KEYS + cdist.MAX_KEYS + ["unique_hist"]:
            assert red[k] == one[k], k
        assert abs(red["sum_sq_err"] - one["sum_sq_err"]) <= 1e-12 * max(1.0, one["sum_sq_err"])
        assert red["max_abs_err"] == one["max_abs_err"]


def test_strip_shards_partition_rows_on_wave_boundaries():
    for hf in (2160, 1080, 42, 5, 3):
        for world in (1, 2, 3, 4, 8):
            spans = [cdist.strip_shard(hf, world, r) for r in range(world)]
            rows = [y for r0, n in spans for y in range(r0, r0 + n)]
            assert rows == list(range(hf))
            assert all(r0 % 4 == 0 for r0, n in spans)
