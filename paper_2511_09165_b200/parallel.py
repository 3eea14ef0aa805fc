"""Direction-grid sharding over GPUs: one process per GPU.

Every pixel (t, psi) is independent (the envelope runs along t within one psi row), so the
direction grid splits into contiguous slices, one per rank.  The exchange itself -- the root's
signals broadcast to every rank and the image shards gathered onto the root, both chunked and
overlapped with the compute -- runs inside libdmas over NCCL (a sharded plan, include/dmas.h
`n_ranks / rank / root / comm_id`).  torch.distributed is only the rendezvous here: rank 0 asks
the library for an NCCL unique id and the process group broadcasts those 128 bytes.  Per-pixel
arithmetic does not depend on the slice, so shards are bitwise the rows a single-GPU plan computes
for the same request (tests/test_gpu_parity.py::test_sharded_plan_one_rank_bitwise).
"""

from __future__ import annotations

from typing import Dict, Optional, Tuple


def partition(n_dirs: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous slice [g0, g1) of `n_dirs` directions for `rank` of `world`; sizes differ by <= 1,
    the first n_dirs % world ranks hold one more.  Same rule as the library's dmas_shard_range
    (tests/test_parallel.py checks they agree)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_dirs, world)
    g0 = rank * base + min(rank, extra)
    return g0, g0 + base + (1 if rank < extra else 0)


def share_comm_id(make_id, group=None, src: int = 0) -> bytes:
    """Rendezvous: rank `src` calls `make_id()` (dmas.comm_id), every rank returns those bytes
    (torch.distributed broadcast_object_list; works on gloo and NCCL process groups)."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


class ShardedBeamformer:
    """One rank's share of a direction-sharded beamformer: a sharded libdmas plan of its slice."""

    def __init__(self, mic_xyz, dir_az_el, fs, c, order, n_samples, *, group=None, device: Optional[int] = None,
                 root: int = 0, **plan_kw):
        import torch
        import torch.distributed as dist
        from . import dmas
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        cid = share_comm_id(dmas.comm_id, group, src=root) if dist.is_initialized() else dmas.comm_id()
        dev = torch.cuda.current_device() if device is None else device
        self.plan = dmas.Plan(mic_xyz, dir_az_el, fs, c, order, n_samples, device=dev, n_ranks=self.world,
                              rank=self.rank, root=root, comm_id=cid, **plan_kw)
        self.g0 = self.plan.dir_begin
        self.g1 = self.g0 + self.plan.n_dirs

    def beamform(self, signals, what: int, gather: bool = False, signals_resident: bool = False,
                 outs=None) -> Dict:
        """A collective: every rank calls it with the same `what`.  `signals` (full shape on every
        rank) is the root's recording, broadcast by the library unless `signals_resident`.  Returns
        this rank's shards, or with `gather` the full images on the root ({} elsewhere)."""
        from . import dmas
        flags = (dmas.GATHER if gather else 0) | (dmas.SIGNALS_RESIDENT if signals_resident else 0)
        return self.plan.beamform(signals, what | flags, outs=outs)

    def close(self):
        self.plan.close()
