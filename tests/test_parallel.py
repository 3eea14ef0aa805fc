"""Multi-rank host logic on CPU: the direction partition, the gather schedule
the library executes over NCCL (checked by simulating every rank's transfer list through the C ABI
on host arrays), the comm-id rendezvous over a world-size-2 gloo process group, and bench.py
spawning its own ranks (`--gpus 2 --dry-run`)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_09165_b200.parallel import partition, share_comm_id

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_partition_covers_exactly():
    for n in (1, 7, 91, 16384, 16385):
        for world in (1, 2, 3, 8):
            if world > n:
                continue
            sl = [partition(n, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [g1 - g0 for g0, g1 in sl]
            assert max(sizes) - min(sizes) <= 1


@pytest.fixture(scope="module")
def dm():
    from paper_2511_09165_b200 import _build
    _build.build()
    from paper_2511_09165_b200 import dmas
    return dmas


def test_library_shard_range_matches_partition(dm):
    for n in (1, 7, 91, 1800, 16384, 16385):
        for world in (1, 2, 3, 5, 8):
            for r in range(world):
                assert dm.shard_range(n, world, r) == partition(n, world, r)


@pytest.mark.parametrize("n_dirs,world,root,F,row", [(16384, 8, 0, 3, 5), (91, 3, 1, 2, 7), (1800, 5, 4, 1, 3),
                                                      (7, 7, 0, 2, 2), (16385, 2, 0, 4, 3), (10, 1, 0, 2, 4)])
def test_gather_schedule_assembles_the_image(dm, n_dirs, world, root, F, row):
    """Run every rank's dmas_gather_schedule on host arrays, pairing each SEND with the RECV the root
    posts for that sender in issue order (NCCL's grouped point-to-point matching rule): the root's
    buffer must come out as the whole image, every element written exactly once, and the shard
    offsets / counts must stay inside their buffers."""
    image = np.arange(F * n_dirs * row, dtype=np.float64).reshape(F, n_dirs, row) + 0.5
    shards, sched = {}, {}
    for r in range(world):
        g0, g1 = dm.shard_range(n_dirs, world, r)
        shards[r] = np.ascontiguousarray(image[:, g0:g1, :]).reshape(-1)
        sched[r] = dm.gather_schedule(n_dirs, world, r, root, F, row)
    dst = np.full(F * n_dirs * row, np.nan)
    hits = np.zeros(F * n_dirs * row, dtype=np.int64)
    recvs = [x for x in sched[root] if x["kind"] == dm.XFER_RECV]
    copies = [x for x in sched[root] if x["kind"] == dm.XFER_COPY]
    assert all(x["kind"] in (dm.XFER_RECV, dm.XFER_COPY) for x in sched[root])
    assert all(x["peer"] == root for x in copies)
    for x in copies:
        assert 0 <= x["src_elem"] and x["src_elem"] + x["count"] <= shards[root].size
        dst[x["dst_elem"]:x["dst_elem"] + x["count"]] = shards[root][x["src_elem"]:x["src_elem"] + x["count"]]
        hits[x["dst_elem"]:x["dst_elem"] + x["count"]] += 1
    for r in range(world):
        if r == root:
            continue
        sends = sched[r]
        assert all(x["kind"] == dm.XFER_SEND and x["peer"] == root for x in sends)
        mine = [x for x in recvs if x["peer"] == r]
        assert len(mine) == len(sends)
        for s, q in zip(sends, mine):                       # matched in issue order
            assert s["count"] == q["count"] and s["frame"] == q["frame"]
            assert 0 <= s["src_elem"] and s["src_elem"] + s["count"] <= shards[r].size
            assert 0 <= q["dst_elem"] and q["dst_elem"] + q["count"] <= dst.size
            dst[q["dst_elem"]:q["dst_elem"] + q["count"]] = shards[r][s["src_elem"]:s["src_elem"] + s["count"]]
            hits[q["dst_elem"]:q["dst_elem"] + q["count"]] += 1
    assert np.all(hits == 1)
    np.testing.assert_array_equal(dst, image.reshape(-1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rendezvous_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cid = share_comm_id(lambda: bytes(range(128)) if rank == 0 else None)
        g = [None] * world
        dist.all_gather_object(g, (rank, cid, partition(16384, world, rank)))
        if rank == 0:
            q.put(g)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_comm_id_rendezvous(world):
    """The sharded plan's rendezvous (parallel.share_comm_id): every rank receives rank 0's id; the
    ranks' slices tile the grid."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rendezvous_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    g = q.get(timeout=5)
    assert [r for r, _, _ in g] == list(range(world))
    assert all(cid == bytes(range(128)) for _, cid, _ in g)
    sl = [s for _, _, s in g]
    assert sl[0][0] == 0 and sl[-1][1] == 16384 and all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


def test_bench_spawns_ranks_dry_run():
    """`bench.py --gpus 2 --dry-run` re-launches itself under torch.distributed.run with 2 ranks
    (gloo, CPU): the line reports n_gpus 2, both ranks, their slices and one shared comm id."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert [x["rank"] for x in line["ranks"]] == [0, 1]
    assert [x["shard"] for x in line["ranks"]] == [[0, 8192], [8192, 16384]]
    assert len({x["comm_id_head"] for x in line["ranks"]}) == 1
    assert len({x["pid"] for x in line["ranks"]}) == 2
    # a mismatched world is refused
    env2 = dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r2 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                        capture_output=True, text=True, timeout=120, env=env2, cwd=ROOT)
    assert r2.returncode != 0
