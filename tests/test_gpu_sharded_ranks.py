"""Direction-sharded plans with 2 and 3 ranks on one GPU, through the library's
in-process loopback transport (include/dmas.h `comm_id` "DMASLOOP"): every rank is a plan of this
process driven from its own thread and CUDA stream, and the exchange the runtime issues -- the
per-chunk broadcast of the root's signals, the chunk agreement, the double-buffered gather staging,
the gather schedule, the host-buffer paths -- runs as event-ordered device copies with NCCL's
matching and completion rules instead of NCCL itself (no kernel ever waits on another rank).

Bar: every rank's shard is bitwise the rows of a single-GPU plan, the gathered images are bitwise
the single-GPU images, and the same holds through dmas_beamform_host, for the root at rank 0 and
at the last rank, with frames split over several exchange chunks."""

import threading

import numpy as np
import pytest

from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dm():
    import torch
    assert torch.cuda.is_available()
    from paper_2511_09165_b200 import dmas
    return dmas


def _run_ranks(world, fn):
    """fn(rank) in `world` threads, each on its own CUDA stream; re-raises the first failure."""
    import torch
    out, errs = [None] * world, []

    def body(r):
        try:
            s = torch.cuda.Stream(device=0)
            with torch.cuda.stream(s):
                out[r] = fn(r)
                s.synchronize()
        except Exception as e:          # noqa: BLE001 -- reported below
            import sys
            import traceback
            print(f"rank {r} failed: {e!r}", file=sys.stderr, flush=True)
            traceback.print_exc()
            errs.append((r, e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
        assert not t.is_alive(), "rank thread hung"
    if errs:
        raise errs[0][1]
    return out


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("world,root", [(2, 0), (3, 0), (3, 2), (8, 5)])
@pytest.mark.parametrize("what_name", ["env_all", "raw_env_mix"])
def test_sharded_ranks_bitwise(dm, world, root, what_name, fused):
    """fused = 1: envelope-only gathers store each rank's rows straight into the root's images from
    the tensor-core envelope kernel (include/dmas.h fused_gather); raw + envelope requests fall back
    to the staged gather."""
    import torch
    cfg = gen.config("C3")
    sig = np.concatenate([cfg["signals"], gen.random_signals(4, 32, cfg["T"], seed=57)])     # 5 frames
    what = (dm.ENV(dm.KIND_ALL) if what_name == "env_all"
            else dm.RAW(dm.KIND_CFDMAS) | dm.ENV(dm.KIND_CFDMAS | dm.KIND_DAS))
    args = (cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 3, cfg["T"])
    plain = dm.Plan(*args, max_frames=5, scratch_bytes=1)             # 1 frame per exchange chunk
    ref = {k: v.cpu().numpy() for k, v in plain.beamform(torch.from_numpy(sig).cuda(), what).items()}
    plain.close()
    cid = dm.loopback_comm_id()
    n_dirs = len(cfg["dirs"])
    plans = _run_ranks(world, lambda r: dm.Plan(*args, max_frames=5, scratch_bytes=1, n_ranks=world, rank=r,
                                                root=root, comm_id=cid, device=0, fused_gather=fused))
    for r, p in enumerate(plans):
        assert p.sharded and p.info["n_dirs_total"] == n_dirs
        assert (p.dir_begin, p.dir_begin + p.n_dirs) == dm.shard_range(n_dirs, world, r)

    def step(r):
        p = plans[r]
        x = torch.from_numpy(sig).cuda() if r == root else torch.zeros(sig.shape, dtype=torch.float32, device="cuda")
        resident = {k: v.cpu().numpy() for k, v in p.beamform(x, what).items()}
        x2 = torch.from_numpy(sig).cuda() if r == root else torch.full(sig.shape, 7.0, device="cuda")
        gathered = {k: v.cpu().numpy() for k, v in p.beamform(x2, what | dm.GATHER).items()}
        host = p.beamform_host(sig if r == root else None, what, n_frames=sig.shape[0])
        host_g = p.beamform_host(sig if r == root else None, what | dm.GATHER, n_frames=sig.shape[0])
        return resident, gathered, host, host_g

    res = _run_ranks(world, step)
    for r, (resident, gathered, host, host_g) in enumerate(res):
        g0, g1 = dm.shard_range(n_dirs, world, r)
        for k in ref:
            assert np.array_equal(resident[k], ref[k][:, g0:g1]), ("resident", r, k)
            assert np.array_equal(host[k], ref[k][:, g0:g1]), ("host shard", r, k)
            if r == root:
                assert np.array_equal(gathered[k], ref[k]), ("gathered", k)
                assert np.array_equal(host_g[k], ref[k]), ("host gathered", k)
        if r != root:
            assert gathered == {} and host_g == {}
    for p in plans:
        p.close()


def test_sharded_rank_failure_is_reported_everywhere(dm):
    """A rank whose plan fails after the communicator is up (here: rank 1 asks for an impossible
    envelope scratch, 5 kinds x 65,535 frames of a C5 image) takes the other ranks down with it
    through the plan-time agreement: every rank returns an error instead of waiting forever."""
    cfg = gen.config("C5", frames=1)
    cid = dm.loopback_comm_id()
    world = 2

    def make(r):
        kw = dict(n_ranks=world, rank=r, root=0, comm_id=cid, device=0, max_frames=1)
        if r == 1:
            kw.update(max_frames=65535, scratch_bytes=1 << 60)
        try:
            dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], **kw)
            return "ok"
        except dm.DmasError as e:
            return (e.status, str(e))

    out = _run_ranks(world, make)
    assert out[1] != "ok" and out[1][0] == 6, out          # DMAS_ERR_OOM on the failing rank
    assert out[0] != "ok" and out[0][0] == 7, out          # DMAS_ERR_NCCL: "another rank failed"
