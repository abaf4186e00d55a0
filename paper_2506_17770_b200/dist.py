"""Multi-GPU driver pieces: frame sharding and the statistics reduction.

The hot path has no data exchange: waves never read another wave's data
and the paper's collaboration is intra-wave only.  So frames are
sharded across ranks with no data-path collective; NCCL (or gloo in the CPU
tests) carries only
  * the max-over-ranks step time, and
  * one all_gather of fixed-size per-rank statistics vectors, reduced in rank
    order on every rank (bitwise identical results for any world size and any
    NCCL reduction order, including the fp64 error sums).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

# integer counters of ctf_frame_stats reduced by sum / max (include/ctf.h)
SUM_KEYS = ["waves_live", "waves_partial", "waves_exact", "waves_fallback", "waves_magnified", "pixels_active",
            "pixels_in_magnified_waves", "texel_evals", "texel_evals_in_magnified_waves", "err_pixels"]
MAX_KEYS = ["max_evals_per_lane", "max_unique_per_wave"]


def frame_shard(total_frames: int, world: int, rank: int) -> range:
    """Contiguous block of frames for `rank` (strong scaling of a fixed batch)."""
    base, extra = divmod(total_frames, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def strip_shard(hf: int, world: int, rank: int) -> tuple[int, int]:
    """Strip sharding of one frame: the ceil(Hf/4) wave-rows are split into
    `world` contiguous strips (sizes differ by at most one wave-row); returns (row0, rows) in
    pixels: rank `rank` filters frame rows [row0, row0 + rows), row0 a multiple of 4 (wave rows
    never straddle two strips, and waves never read another wave's pixels)."""
    wr = frame_shard((hf + 3) // 4, world, rank)
    row0 = 4 * wr.start
    return row0, max(0, min(4 * wr.stop, hf) - row0)


def weak_frames(frames_per_rank: int, rank: int, period: int = 64) -> tuple[list[int], int]:
    """Weak scaling: rank r filters its own frames_per_rank frames of the camera path
    (path position f mod period) with distinct RNG frame indices starting at r*frames_per_rank."""
    first = rank * frames_per_rank
    return [(first + f) % period for f in range(frames_per_rank)], first


def _pack(st: dict) -> tuple[torch.Tensor, torch.Tensor]:
    ints = [int(st[k]) for k in SUM_KEYS + MAX_KEYS] + [int(x) for x in st["unique_hist"]]
    flts = [float(st.get("sum_sq_err", 0.0)), float(st.get("max_abs_err", 0.0))]
    return torch.tensor(ints, dtype=torch.int64), torch.tensor(flts, dtype=torch.float64)


def _unpack(ints: torch.Tensor, flts: torch.Tensor) -> dict:
    v = ints.tolist()
    n = len(SUM_KEYS) + len(MAX_KEYS)
    st = dict(zip(SUM_KEYS + MAX_KEYS, v[:n]))
    st["unique_hist"] = v[n:]
    st["sum_sq_err"], st["max_abs_err"] = flts.tolist()
    return st


def reduce_stats_local(per_rank: list[dict]) -> dict:
    """Rank-ordered reduction of a list of stats dicts (the definition all ranks apply)."""
    out = {k: 0 for k in SUM_KEYS}
    out.update({k: 0 for k in MAX_KEYS})
    out["unique_hist"] = [0] * 129
    out["sum_sq_err"], out["max_abs_err"] = 0.0, 0.0
    for st in per_rank:
        for k in SUM_KEYS:
            out[k] += int(st[k])
        for k in MAX_KEYS:
            out[k] = max(out[k], int(st[k]))
        out["unique_hist"] = [a + int(b) for a, b in zip(out["unique_hist"], st["unique_hist"])]
        out["sum_sq_err"] += float(st.get("sum_sq_err", 0.0))
        out["max_abs_err"] = max(out["max_abs_err"], float(st.get("max_abs_err", 0.0)))
    return out


def reduce_stats(st: dict, device: torch.device | str = "cpu", group=None) -> dict:
    """all_gather every rank's stats vector, then reduce in rank order (deterministic)."""
    if not dist.is_available() or not dist.is_initialized():
        return reduce_stats_local([st])
    ws = dist.get_world_size(group)
    ints, flts = _pack(st)
    ints, flts = ints.to(device), flts.to(device)
    gi = [torch.empty_like(ints) for _ in range(ws)]
    gf = [torch.empty_like(flts) for _ in range(ws)]
    dist.all_gather(gi, ints, group=group)
    dist.all_gather(gf, flts, group=group)
    return reduce_stats_local([_unpack(a.cpu(), b.cpu()) for a, b in zip(gi, gf)])


def reduce_frame_stats(records: list[dict], group=None) -> dict:
    """Whole-job statistics from per-frame records: every rank contributes the
    stats of the frames (or frame strips) it filtered, each tagged with 'frame' and 'row0'; the
    records of all ranks are gathered (all_gather_object) and reduced on every rank in global
    (frame, row0) order.  With frame sharding the reduction therefore sees exactly the records,
    in exactly the order, of a 1-GPU run: every total, including the fp64 error sums, is
    bitwise independent of the number of GPUs.  With strip sharding the integer totals are
    bitwise identical too; the fp64 error sums of a frame are the sum of its strips' sums."""
    items = list(records)
    if dist.is_available() and dist.is_initialized():
        ws = dist.get_world_size(group)
        gathered = [None] * ws
        dist.all_gather_object(gathered, items, group=group)
        items = [r for part in gathered for r in part]
    items.sort(key=lambda r: (int(r["frame"]), int(r.get("row0", 0))))
    return reduce_stats_local(items)


def sum_over_ranks(x: int, device: torch.device | str = "cpu", group=None) -> int:
    if not dist.is_available() or not dist.is_initialized():
        return int(x)
    t = torch.tensor([int(x)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def max_over_ranks(x: float, device: torch.device | str = "cpu", group=None) -> float:
    if not dist.is_available() or not dist.is_initialized():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
