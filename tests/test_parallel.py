"""Multi-rank host logic on CPU (gloo, world_size 2): direction partition, signal broadcast,
shard gather and reassembly.  The per-shard compute here is the oracle (tests may call it);
on GPUs the same helpers move the CUDA plan's shards."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_09165_b200.parallel import gather_shards, partition, broadcast_signals


def test_partition_covers_exactly():
    for n in (1, 7, 91, 16384, 16385):
        for world in (1, 2, 3, 8):
            sl = [partition(n, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [g1 - g0 for g0, g1 in sl]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import dmas_oracle as O
        from workloads import gen
        cfg = gen.config("C1")
        n_dirs = len(cfg["dirs"])
        # rank 0 owns the recording; the others receive it by broadcast
        x = torch.from_numpy(cfg["signals"]) if rank == 0 else torch.zeros(cfg["signals"].shape, dtype=torch.float32)
        broadcast_signals(x, src=0)
        g0, g1 = partition(n_dirs, world, rank)
        d = O.delay_table(cfg["mic_xyz"], cfg["dirs"][g0:g1], cfg["fs"], cfg["c"])
        img = O.beamform_frame(x.numpy()[0], d, cfg["order"])["cfdmas"]
        full = gather_shards(torch.from_numpy(img[None]), n_dirs, dst=0)
        if rank == 0:
            d_all = O.delay_table(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"])
            ref = O.beamform_frame(cfg["signals"][0], d_all, cfg["order"])["cfdmas"]
            q.put(float(np.max(np.abs(full.numpy()[0] - ref))) / float(np.max(np.abs(ref))))
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_broadcast_shard_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) <= 1e-12
