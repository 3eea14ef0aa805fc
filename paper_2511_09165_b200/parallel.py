"""Direction-grid sharding over GPUs: one process per GPU, torch.distributed (NCCL) plumbing.

Every pixel (t, psi) is independent (the envelope runs along t within one psi row), so the
direction grid splits into contiguous slices, one per rank.  Each rank builds
its own plan (its slice of the delay table), receives the whole signal block by one broadcast
from the source rank, beamforms its slice, and the image shards are either kept resident or
gathered to one rank along the direction axis.  Per-pixel arithmetic does not depend on the
slice, so the assembled images are bitwise identical to a single-GPU run (tested in
tests/test_gpu_parity.py::test_chunking_and_sharding_bitwise).

The collective helpers are backend-agnostic (they run on gloo/CPU in tests/test_parallel.py);
the compute is always the CUDA plan — there is no CPU path here.
"""

from __future__ import annotations

from typing import Dict, Optional, Tuple


def partition(n_dirs: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous slice [g0, g1) of `n_dirs` directions for `rank` of `world`; sizes differ by <= 1."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_dirs, world)
    g0 = rank * base + min(rank, extra)
    return g0, g0 + base + (1 if rank < extra else 0)


def broadcast_signals(x, src: int = 0, group=None):
    """Broadcast the [F][n_mics][T] signal block from `src` to every rank (in place)."""
    import torch.distributed as dist
    dist.broadcast(x, src=src, group=group)
    return x


def gather_shards(shard, n_dirs: int, dst: int = 0, group=None):
    """Gather per-rank image shards [F][n_dirs_g][T'] along the direction axis onto `dst`.

    Shards may differ in size by one row (see `partition`); they are padded to the largest
    shard for the collective and trimmed on assembly.  Returns the full [F][n_dirs][T'] tensor
    on `dst` and None elsewhere."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    F, _, Tp = shard.shape
    rows = [partition(n_dirs, world, r) for r in range(world)]
    mx = max(g1 - g0 for g0, g1 in rows)
    padded = torch.zeros((F, mx, Tp), dtype=shard.dtype, device=shard.device)
    padded[:, :shard.shape[1]] = shard
    bufs = [torch.empty_like(padded) for _ in range(world)] if rank == dst else None
    if dist.get_backend(group) == "nccl":
        # NCCL has no gather; all_gather into the list (every rank receives; non-dst ranks discard)
        bufs = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(bufs, padded, group=group)
    else:
        dist.gather(padded, gather_list=bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:, :g1 - g0] for b, (g0, g1) in zip(bufs, rows)], dim=1)


class ShardedBeamformer:
    """One rank's share of a direction-sharded beamformer (the CUDA plan of its slice)."""

    def __init__(self, mic_xyz, dir_az_el, fs, c, order, n_samples, *, group=None, device: Optional[int] = None,
                 **plan_kw):
        import torch
        import torch.distributed as dist
        from . import dmas
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n_dirs = len(dir_az_el)
        self.g0, self.g1 = partition(self.n_dirs, self.world, self.rank)
        dev = torch.cuda.current_device() if device is None else device
        self.plan = dmas.Plan(mic_xyz, dir_az_el[self.g0:self.g1], fs, c, order, n_samples, device=dev, **plan_kw)

    def beamform(self, signals, what: int, src: Optional[int] = 0, gather_to: Optional[int] = None) -> Dict:
        """Broadcast `signals` from `src` (None: every rank already holds them), beamform this
        rank's slice, and optionally gather every image to rank `gather_to`."""
        if src is not None and self.world > 1:
            broadcast_signals(signals, src, self.group)
        res = self.plan.beamform(signals, what)
        if gather_to is None or self.world == 1:
            return res
        return {k: gather_shards(v, self.n_dirs, gather_to, self.group) for k, v in res.items()}

    def close(self):
        self.plan.close()
