#!/usr/bin/env python
"""Throughput benchmark of the DMAS / CF beamforming hot path on B200.

Metric (BASELINE.json): "CF-DMAS images/sec (directions x range samples per second)", i.e.
pixels/s = frames * n_dirs * T / time.  Workload: BASELINE.json configs[4] = C5, the streaming
config the metric's 1/2/4/8-GPU throughput is quoted on: 32-mic eRTIS-like
array, 16,384 directions (128 az x 128 el), T = 4096 at 450 kHz, 256 frames per step, CF-DMAS
p = 2 followed by the 127-tap 5 kHz envelope.  One step = one dmas_beamform call over the
256-frame batch (every §8(a) row: signed roots -> gather / power sums / Newton-Girard / CF ->
envelope); the delay table (A1) is built once per plan, as the paper pre-computes it.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path, one process per GPU
  python bench.py --impl reference ...                      # the float64 oracle on the host cores
  python bench.py --gpus 2 --dry-run                        # CPU: rank spawning / sharding only

Multi-GPU (north_star, default `--mode dirshard`): the direction grid is split
into contiguous slices, one per rank; each step the root's 256-frame recording is broadcast and
every rank beamforms its slice -- both inside libdmas (a sharded plan, NCCL), the broadcast of
frame chunk c + 1 overlapped with the compute of chunk c.  `value` keeps the image shards resident
(the units all ranks processed / the max over ranks of the step time: strong scaling, the total
work is fixed); the line's `gathered` object times the same step with every image gathered onto
the root (grouped send / recv per chunk, overlapped with the next chunk).  `--mode weak` instead
gives every rank its own 256-frame stream over the whole grid (replicas, no exchange).
With `--gpus N` and no torchrun environment, the script re-launches itself under
torch.distributed.run with N ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import gen  # noqa: E402

METRIC = "CF-DMAS images/sec (directions x range samples per second) at 1/2/4/8 B200"
UNIT = "px/s"
LP_TAPS = 127
FP32_LANES_PER_SM_CLK = 128     # FFMA/FADD/FMUL lanes per SM per clock (guide; tools/ubench_fp32.cu measures it)
# SURVEY.md §8(d) FLOP convention (FADD/FMUL = 1, FFMA = 2): algorithmic FLOP per pixel of the
# beamform = N_m * phi_p + 30, phi_p = 5 / 6 / 9 / 10 for p = 2 / 3 / 4 / 5
PHI_P = {2: 5, 3: 6, 4: 9, 5: 10}
# FP32-pipe lane-ops per microphone sample of k_beamform_lds64 as issued and per pixel epilogue
OPS_PER_MIC = {2: 5, 3: 6, 4: 9, 5: 9}
OPS_EPI = {2: 6, 3: 10, 4: 14, 5: 18}
BF_KERNELS = {0: "k_beamform", 1: "k_beamform_lds64", 2: "k_beamform_mg"}   # dmas_plan_info.bf_kernel
SURVEY_F2_CEILING = {"C5": 131e9 / 1e9, "C4": 73e9 / 1e9}    # SURVEY.md §8(d) model ceilings, Gpx/s per GPU
ENV_PRECISION = ("tcgen05 low-pass, 3-pass BF16 split: <= 3 * 2^-16 ~ 4.6e-5 of the envelope value (bound); "
                 "the FP32 FIR (env_engine = 1) is timed in all_fp32")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=0, help="frames per step (0: the workload's, C5 256, C4 16)")
    ap.add_argument("--workload", choices=["C5", "C4"], default="C5",
                    help="C5 = the metric's config (default); C4 = 64-mic p = 3 secondary line")
    ap.add_argument("--mode", choices=["dirshard", "weak"], default="dirshard")
    ap.add_argument("--bf-engine", type=int, choices=[0, 1], default=0,
                    help="beamform kernel: 0 auto (LDS.64 kernel where it fits), 1 classic k_beamform (comparison)")
    ap.add_argument("--env-engine", type=int, choices=[0, 1, 2], default=0,
                    help="envelope low-pass: 0 tcgen05 (BF16 split written by the beamform), 1 the FP32 FIR, "
                         "2 tcgen05 on the fp32 image (split inside the envelope kernel; comparison)")
    ap.add_argument("--interp", action="store_true",
                    help="linear-interpolation pre-steering (fractional delays, roots on the fly; NEXT-2)")
    ap.add_argument("--raw", action="store_true",
                    help="raw recordings in: the step includes the GPU matched filter (paper Fig. 1 pipeline)")
    ap.add_argument("--e2e-frames", type=int, default=0, help="frames per e2e step (0: the whole step)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip all_fp32 / linearity / C1 latency")
    ap.add_argument("--cpu-dirs", type=int, default=0, help="directions per core in the all-core CPU sample (0 = all)")
    ap.add_argument("--dry-run", action="store_true", help="CPU only: spawn ranks, shard the grid, print the line")
    ap.add_argument("--fused-gather", action="store_true",
                    help="sharded plans: the gathered step stores each rank's envelope rows straight into the "
                         "root's image (include/dmas.h fused_gather) instead of staged send / recv")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use a sharded plan (NCCL communicator, broadcast, gather) even on one GPU: exercises "
                         "the multi-GPU code path of this script and the library where only one GPU is available")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


_OUT = sys.stdout


def emit(line: dict):
    """The one JSON line of the run, on the real stdout."""
    _OUT.write(json.dumps(line) + "\n")
    _OUT.flush()


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int) -> int:
    """--gpus N without a torchrun environment: re-launch this script with N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def _oracle_chunk(job):
    from oracle import dmas_oracle as O
    sig, d, p = job
    h = O.lpf_taps(LP_TAPS, 5000.0, gen.FS)
    img = O.beamform_frame(sig, d, p)
    e = O.envelope(img["cfdmas"], h)
    return e.shape[0] * e.shape[1]


def oracle_rate(cfg, n_dirs, cores, pool=None, frame_idx=0):
    """Time the float64 oracle (as it stands) on a bounded sample of the step: one frame, `n_dirs`
    directions spread over the grid, all T samples, CF-DMAS + envelope, split over `cores`
    processes (contiguous direction chunks).  The delay table is built outside the timed region,
    as in the CUDA path's plan.  Returns (px/s, seconds, px)."""
    import multiprocessing as mp
    from oracle import dmas_oracle as O
    n = min(len(cfg["dirs"]), n_dirs)
    sel = np.linspace(0, len(cfg["dirs"]) - 1, n).astype(int)
    d = O.delay_table(cfg["mic_xyz"], cfg["dirs"][sel], cfg["fs"], cfg["c"])
    dpc = -(-n // cores)
    jobs = [(cfg["signals"][frame_idx], d[i:i + dpc], cfg["order"]) for i in range(0, n, dpc)]
    if cores == 1:
        t0 = time.perf_counter()
        px = sum(_oracle_chunk(j) for j in jobs)
        dt = time.perf_counter() - t0
        return px / dt, dt, px
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
    try:
        t0 = time.perf_counter()
        px = sum(pool.map(_oracle_chunk, jobs))
        dt = time.perf_counter() - t0
    finally:
        if own:
            pool.close()
            pool.join()
    return px / dt, dt, px


def cpu_baseline(args):
    """The oracle on this host (SURVEY.md §8(d) "Oracle"): all cores over one whole frame, one
    process over 1024 directions, and the linearity check of PAPER.md:284 (time proportional to
    the number of directions) on one process at 128 / 256 / 512 directions."""
    cfg = gen.config(args.workload, frames=1)
    cores = os.cpu_count() or 1
    n_all = len(cfg["dirs"]) if not args.cpu_dirs else cores * args.cpu_dirs
    r_all, dt_all, px_all = oracle_rate(cfg, n_all, cores)
    r_one, dt_one, px_one = oracle_rate(cfg, 1024, 1)
    lin = {"n_dirs": [], "seconds": [], "px_per_s": []}
    for n in (128, 256, 512):
        r, dt, _ = oracle_rate(cfg, n, 1)
        lin["n_dirs"].append(n)
        lin["seconds"].append(dt)
        lin["px_per_s"].append(r)
    lin["time_ratio_512_vs_128"] = lin["seconds"][2] / lin["seconds"][0]
    return {"value": r_all, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"frame 0 of {cfg['name']}: {n_all} of {len(cfg['dirs'])} directions x {cfg['T']} samples = "
                       f"{px_all} px, CF-DMAS p={cfg['order']} + {LP_TAPS}-tap envelope, float64 numpy oracle, "
                       f"{cores} processes; {dt_all:.1f} s"),
            "cpu_model": cpu_model(),
            "single_process": {"value": r_one, "unit": UNIT, "cores": 1,
                               "sample": f"frame 0, 1024 directions spread over the grid = {px_one} px; {dt_one:.1f} s"},
            "linearity": lin}


def run_reference(args, rank, world):
    """The reference arm: the oracle, as it stands, on the host cores (rank 0 only).  Each step
    beamforms one whole frame of the workload (a bounded sample of the 256-frame step) with a
    process pool over all cores; value = median px/s over the timed steps, ms_per_step = the
    measured time of one such step."""
    import multiprocessing as mp
    if rank != 0:
        return 0
    cfg = gen.config(args.workload, frames=1)
    cores = os.cpu_count() or 1
    n_dirs = len(cfg["dirs"]) if not args.cpu_dirs else cores * args.cpu_dirs
    rates, secs, px = [], [], 0
    with mp.get_context("fork").Pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            r, dt, px = oracle_rate(cfg, n_dirs, cores, pool)
            if i >= args.warmup:
                rates.append(r)
                secs.append(dt)
    value = statistics.median(rates)
    sample = (f"each step: frame 0 of {cfg['name']}, {n_dirs} directions x {cfg['T']} samples = {px} px "
              f"(one frame of the {args.frames}-frame step), CF-DMAS p={cfg['order']} + {LP_TAPS}-tap envelope, "
              f"float64 numpy oracle, {cores} processes")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "strong" if args.mode == "dirshard" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded eRTIS-like point-reflector echoes, matched-filtered; workloads/gen.py)",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "ms_per_step is the measured time of one sample step (one frame, all directions); value is px/s "
                "of that sample, the same metric and unit as the GPU arm",
    }
    emit(line)
    return 0


def load_profile():
    """Per-kernel ncu figures from the committed `ncu --set full` capture (profiles/traffic.json:
    dram__bytes_read.sum + dram__bytes_write.sum per launch, FMA-pipe and issue-slot activity)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except OSError:
        return {}


WORKLOADS = {
    "C5": {"array": "32-mic eRTIS-like disk (10 cm)", "n_dirs": 16384, "grid": "128 az (+-90) x 128 el (+-60)",
           "n_samples": 4096, "fs_hz": 450000, "order": 2, "frames": 256,
           "l2": "inputs 128 MiB/GPU > 126 MB L2 and every step streams 64 GiB of output (no L2 reuse across steps)"},
    "C4": {"array": "64-mic disk (10 cm)", "n_dirs": 16384, "grid": "128 az (+-90) x 128 el (+-60)",
           "n_samples": 8192, "fs_hz": 450000, "order": 3, "frames": 16,
           "l2": "every step streams 8 GiB of output (no L2 reuse across steps)"},
}


def config_dict(args, world):
    """The workload; identical for both arms."""
    w = WORKLOADS[args.workload]
    return {"workload": args.workload, "array": w["array"], "n_dirs": w["n_dirs"], "grid": w["grid"],
            "n_samples": w["n_samples"], "fs_hz": w["fs_hz"], "order": w["order"],
            "frames_per_step": args.frames,
            "outputs": f"CF-DMAS{w['order']} envelope (127-tap 5 kHz low-pass)",
            "mode": args.mode, "world": world, "l2": w["l2"],
            "input": "raw recordings, matched filter on the GPU (1125-tap chirp)" if args.raw
                     else "matched-filtered signals (north_star input)",
            "presteer": "linear interpolation (fractional delays)" if args.interp else "nearest sample (integer LUT)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines()]
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9 and r[0].strip() == str(self.idx)]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


def physical_gpu_index(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local < len(ids) and ids[local].strip().isdigit():
            return int(ids[local])
    return local


def step_stats(ms_list):
    s = sorted(ms_list)
    p90 = s[min(len(s) - 1, int(round(0.9 * (len(s) - 1))))]
    return {"median": statistics.median(s), "min": s[0], "p90": p90, "max": s[-1], "n": len(s)}


# ------------------------------------------------------------------ dry run (CPU: spawning / sharding)
def run_dry(args, rank, world):
    import torch.distributed as dist
    from paper_2511_09165_b200 import parallel
    if world > 1:
        dist.init_process_group("gloo")
    n_dirs = WORKLOADS[args.workload]["n_dirs"]
    g0, g1 = parallel.partition(n_dirs, world, rank)
    cid = parallel.share_comm_id(lambda: os.urandom(128)) if world > 1 else os.urandom(128)
    info = {"rank": rank, "shard": [g0, g1], "comm_id_head": cid[:8].hex(), "pid": os.getpid()}
    seen = [None] * world
    if world > 1:
        dist.all_gather_object(seen, info)
    else:
        seen = [info]
    if rank == 0:
        emit({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "dry_run": True,
                          "ranks": seen, "config": config_dict(args, world)})
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local):
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)

    import torch
    import torch.distributed as dist
    from paper_2511_09165_b200 import dmas, parallel

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    sharded = args.mode == "dirshard" and (world > 1 or args.force_sharded)

    # ---- inputs (resident in HBM before the timed region)
    F = args.frames
    if args.raw:
        cfg = gen.raw_config(args.workload, frames=F)
    elif args.mode == "weak":
        cfg = gen.config(args.workload, frames=F, stream=rank)
    else:
        cfg = gen.config(args.workload, frames=F if rank == 0 else 1)   # the recording lives on the root
    dirs, T, p = cfg["dirs"], cfg["T"], cfg["order"]
    n_mics = cfg["mic_xyz"].shape[0]
    x = torch.empty((F,) + cfg["signals"].shape[1:], dtype=torch.float32, device=dev)
    if rank == 0 or not sharded:
        x.copy_(torch.from_numpy(cfg["signals"]))
    kw = dict(max_frames=F, lp_taps=LP_TAPS, mf_coeffs=cfg.get("chirp") if args.raw else None,
              delay_interp=1 if args.interp else 0, bf_engine=args.bf_engine, env_engine=args.env_engine)
    if sharded:
        sb = parallel.ShardedBeamformer(cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], p, T, device=local,
                                        fused_gather=1 if args.fused_gather else 0, **kw)
        plan = sb.plan
    else:
        plan = dmas.Plan(cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], p, T, device=local, **kw)
    bf_name = BF_KERNELS[plan.info["bf_kernel"]]
    what = dmas.ENV(dmas.KIND_CFDMAS)
    out = torch.empty((F, plan.n_dirs, T), dtype=torch.float32, device=dev)    # this rank's rows
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def timed_steps(fn, n):
        """n steps bracketed by a barrier + synchronize on both sides; per-step CUDA events on the
        launching stream; returns (total ms max over ranks, per-step ms of this rank)."""
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        evs[0].record(stream)
        for i in range(n):
            fn()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(n)]
        total = evs[0].elapsed_time(evs[-1])
        if world > 1:
            t = torch.tensor([total], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        barrier()
        return total, per

    def step():
        plan.beamform(x, what, outs=[out])     # sharded: broadcast from the root inside, shards resident

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(physical_gpu_index(local))
    time.sleep(0.3)
    plan.set_timing(True)
    n_launch0 = dmas.launch_count()
    total_ms, per_ms = timed_steps(step, args.steps)
    launches = dmas.launch_count() - n_launch0
    plan.set_timing(False)
    ktime = plan.timing_read()
    clk = clocks.stop()
    ms = total_ms / args.steps
    n_dirs_total = len(dirs)
    px_step = F * n_dirs_total * T * (world if args.mode == "weak" else 1)
    value = px_step / (ms * 1e-3)

    # ---- roofline of the dominant kernel (device time inside the timed region, this rank)
    bf_ms, bf_n = ktime["beamform"]
    env_ms, env_n = ktime["envelope"]
    rt_ms, rt_n = ktime["signed_roots"]
    px_rank = F * plan.n_dirs * T
    px_launch_bf = px_rank / max(1, bf_n / args.steps)
    px_launch_env = px_rank / max(1, env_n / args.steps)
    bf_avg = bf_ms / max(1, bf_n)
    env_avg = env_ms / max(1, env_n)
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = (clk or {}).get("sm_max_mhz") or 1965.0
    lane_peak = FP32_LANES_PER_SM_CLK * sm_count * sm_max * 1e6 / 1e12      # T lane-ops/s at max clock
    flop_peak = 2.0 * lane_peak                                            # TFLOP/s, FFMA = 2
    flop_px = n_mics * PHI_P[p] + 30                                        # SURVEY §8(d), beamform only
    ach_flop = flop_px * px_launch_bf / (bf_avg * 1e-3) / 1e12
    ops_px = OPS_PER_MIC[p] * n_mics + OPS_EPI[p]
    ach_ops = ops_px * px_launch_bf / (bf_avg * 1e-3) / 1e12
    hbm_peak = 6547.2
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    env_gbs = 8.0 * px_launch_env / (env_avg * 1e-3) / 1e9 if env_n else 0.0   # read raw + write envelope
    prof = load_profile()
    frames_launch = F / max(1, bf_n / args.steps)
    pb = prof.get("k_beamform", {})
    traffic_launch = (pb["dram_bytes_per_launch"] * frames_launch / pb["frames_per_launch"]
                      if pb.get("dram_bytes_per_launch") and pb.get("frames_per_launch") else None)
    roofline = {
        "bound": "alu", "kernel": bf_name, "achieved": ach_flop, "peak": flop_peak,
        "unit": "TFLOP/s (FP32, FFMA = 2)", "frac": ach_flop / flop_peak, "traffic": traffic_launch,
        "traffic_unit": "bytes per launch (ncu dram read+write, scaled to this launch's frames)",
        "algorithmic_bytes": 4.0 * px_launch_bf,
        "flop_per_px": flop_px,
        "flop_basis": f"SURVEY.md §8(d): N_m * phi_p + 30 = {n_mics} * {PHI_P[p]} + 30 (FADD/FMUL = 1, FFMA = 2)",
        "peak_basis": (f"{FP32_LANES_PER_SM_CLK} FP32 lanes/clk/SM x 2 x {sm_count} SMs x {sm_max:.0f} MHz "
                       "(guide unit counts at the max SM clock; tools/ubench_fp32.cu measures lanes/clk, "
                       "profiles/r02/ubench.json)"),
        "step_s8d": {"flop_per_px": flop_px + 2 * LP_TAPS, "TFLOP_s": (flop_px + 2 * LP_TAPS) * value / 1e12,
                     "frac": (flop_px + 2 * LP_TAPS) * value / 1e12 / (flop_peak * world),
                     "model_ceiling_gpx_s": SURVEY_F2_CEILING.get(args.workload),
                     "note": "SURVEY.md §8(d) whole-step count N_m*phi_p + 30 + 254 per enveloped image (the "
                             "127-tap low-pass as FP32 FMAs, although it runs on the tensor cores) against the "
                             "FP32 peak of all GPUs; model_ceiling = the §8(d) F2 ceiling of the step (Gpx/s, 1 GPU)"},
        "issue": {"lane_ops_per_px": ops_px, "T_lane_ops_s": ach_ops, "frac_of_lane_peak": ach_ops / lane_peak,
                  "formulation_flop_ceiling": PHI_P[p] / (2.0 * OPS_PER_MIC[p]),
                  "ncu_fma_pipe_pct": pb.get("pipe_fma_pct"), "ncu_issue_active_pct": pb.get("issue_active_pct"),
                  "note": "the kernel issues 5 FP32 instructions per mic-pixel at p = 2 (x = s|s| is recomputed "
                          "from the one staged root plane), of which the §8(d) count credits 5 FLOP: its FLOP "
                          "fraction cannot exceed phi_p / (2 * ops) = 0.5"},
        "kernels": {
            "beamform": {"avg_ms": bf_avg, "launches": bf_n, "share": bf_ms / total_ms,
                         "Gpx_s": px_launch_bf / (bf_avg * 1e-3) / 1e9, "TFLOP_s": ach_flop,
                         "frac": ach_flop / flop_peak},
            "envelope": {"avg_ms": env_avg, "launches": env_n, "share": env_ms / total_ms, "bound": "hbm",
                         "GB_s": env_gbs, "hbm_frac": env_gbs / hbm_peak, "algorithmic_bytes_per_px": 8,
                         "Gpx_s": px_launch_env / (env_avg * 1e-3) / 1e9 if env_n else None,
                         "engine": "FP32 FIR" if args.env_engine == 1 else "tcgen05 BF16x3" + (
                             " (fp32 input, in-kernel split)" if args.env_engine == 2 else " (pre-split input)"),
                         "ncu_dram_bytes_per_launch": prof.get("k_envelope", {}).get("dram_bytes_per_launch"),
                         "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"},
            "signed_roots": {"avg_ms": rt_ms / max(1, rt_n), "launches": rt_n, "share": rt_ms / total_ms}}}

    # ---- sharded: the same step with every image gathered onto the root (overlapped per chunk)
    gathered = None
    if sharded:
        out_full = torch.empty((F, n_dirs_total, T), dtype=torch.float32, device=dev) if rank == 0 else None

        def step_g():
            plan.beamform(x, what | dmas.GATHER, outs=[out_full] if rank == 0 else None)

        step_g()
        ng = max(1, min(args.steps, 3))
        tg, per_g = timed_steps(step_g, ng)
        gathered = {"value": px_step / (tg / ng * 1e-3), "unit": UNIT, "ms_per_step": tg / ng, "steps": ng,
                    "gather_bytes_to_root_per_step": int(F * (n_dirs_total - plan.n_dirs) * T * 4),
                    "fused": bool(args.fused_gather),
                    "note": ("fused: every rank's tensor-core envelope stores its rows straight into the root's "
                             "image (CUDA IPC mapping, TMA stores), then a stream-ordered barrier"
                             if args.fused_gather else
                             "broadcast + compute + grouped ncclSend/ncclRecv of every chunk's shards into the "
                             "root's image, overlapped with the next chunk; root link-bound")}
        del out_full

    # ---- end to end through the public API with host buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e and not args.raw:
        Fe = min(args.e2e_frames or F, F)
        # every rank lands its own image rows in host memory (sharded: its shard, copied over its
        # own PCIe link; the root's recording comes in and is broadcast on the device)
        rows_h = plan.n_dirs
        try:                                              # the whole step: 64 GiB of pinned images for C5
            hout = torch.empty((Fe, rows_h, T), dtype=torch.float32, pin_memory=True)
        except RuntimeError:
            Fe = min(16, F)
            hout = torch.empty((Fe, rows_h, T), dtype=torch.float32, pin_memory=True)
        if world > 1:                                     # every rank takes the smallest Fe
            t = torch.tensor([Fe], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            Fe = int(t.item())
            hout = hout[:Fe]
        hsig = None
        if rank == 0 or not sharded:
            hsig = torch.empty((Fe,) + cfg["signals"].shape[1:], dtype=torch.float32, pin_memory=True)
            hsig.copy_(torch.from_numpy(cfg["signals"][:Fe]))

        def call_host():
            if hsig is not None:
                plan.beamform_host(hsig.numpy(), what, outs=[hout.numpy()])
            else:
                plan.beamform_host(None, what, outs=[hout.numpy()], n_frames=Fe)

        call_host()                                   # warm-up (allocates the staging)
        times = []
        for _ in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            call_host()
            times.append(time.perf_counter() - t0)
        et = statistics.median(times)
        if world > 1:
            t = torch.tensor([et], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e_px = Fe * n_dirs_total * T * (world if args.mode == "weak" else 1)
        e2e = {"value": e_px / et, "unit": UNIT,
               "h2d_bytes_per_step": int(Fe * n_mics * T * 4) * (world if args.mode == "weak" else 1),
               "d2h_bytes_per_step": int(e_px * 4), "frames_per_step": Fe,
               "ratio_to_device_value": (e_px / et) / value, "seconds_per_step": et,
               "timing": "host wall clock around the synchronous dmas_beamform_host call, max over ranks (pinned "
                         "host buffers; H2D, kernels and D2H pipelined in chunks; sharded: the root's recording in, "
                         "broadcast on the device, every rank's image shard out over its own PCIe link); bound by "
                         "the PCIe device-to-host copy of fp32 images"}

    # ---- extras on one GPU: all-FP32 step, linearity in N_psi, C1 launch latency
    extras = {}
    if rank == 0 and world == 1 and not args.no_extras and not args.raw:
        extras = gpu_extras(args, cfg, plan, x, out, kw, dmas, torch, dev, stream, value)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if args.mode == "dirshard" else "weak", "vs_baseline": None,
            "dtype": "f32" + ("" if args.env_engine == 1 else "+bf16x3(tcgen05 envelope)"),
            "dtype_detail": ("beamform A2-A4 in FP32 (delay table A1 in FP64); " +
                             ("envelope FP32 FIR" if args.env_engine == 1 else ENV_PRECISION)),
            "data": "synthetic (seeded eRTIS-like point-reflector echoes, matched-filtered; workloads/gen.py)",
            "config": config_dict(args, world), "beamform_kernel": bf_name,
            "frames_per_s": F * (world if args.mode == "weak" else 1) / (ms * 1e-3),
            "step_ms": step_stats(per_ms),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        if gathered:
            line["gathered"] = gathered
        line.update(extras)
        if e2e and extras.get("pcie_d2h_GB_s"):
            e2e["d2h_GB_s"] = e2e["d2h_bytes_per_step"] / e2e["seconds_per_step"] / 1e9
            e2e["frac_of_measured_pcie_d2h"] = e2e["d2h_GB_s"] / extras["pcie_d2h_GB_s"]
        emit(line)
    if sharded:
        sb.close()
    else:
        plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def gpu_extras(args, cfg, plan, x, out, kw, dmas, torch, dev, stream, value):
    """(1) the same step with the FP32 FIR envelope (env_engine = 1: every multiply FP32);
    (2) time against N_psi on the GPU ("linear"): the first 4096 / 8192 / 16384
    directions, 64 frames; (3) C1 (BASELINE configs[0], 93 k pixels per frame: launch-latency
    bound) per-frame latency, eager calls vs one CUDA-graph replay of 100 single-frame calls."""
    F, T, p = x.shape[0], cfg["T"], cfg["order"]
    what = dmas.ENV(dmas.KIND_CFDMAS)
    res = {}

    def time_fn(fn, n, warm=1):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    if args.env_engine == 0:
        p32 = dmas.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], p, T, device=dev.index,
                        **dict(kw, env_engine=1))
        ms32 = time_fn(lambda: p32.beamform(x, what, outs=[out]), 3)
        res["all_fp32"] = {"value": F * len(cfg["dirs"]) * T / (ms32 * 1e-3), "unit": UNIT, "ms_per_step": ms32,
                           "steps": 3, "env_engine": 1,
                           "note": "same step, envelope low-pass as the FP32 FIR (k_envelope_lp127): no BF16 anywhere"}
        p32.close()

    lin = {"n_dirs": [], "ms": [], "px_per_s": [], "frames": 64}
    flat = out.view(-1)
    for n in (4096, 8192, 16384):
        pl = dmas.Plan(cfg["mic_xyz"], cfg["dirs"][:n], cfg["fs"], cfg["c"], p, T, device=dev.index,
                       **dict(kw, max_frames=64))
        o = flat[:64 * n * T].view(64, n, T)
        xs = x[:64]
        t = time_fn(lambda: pl.beamform(xs, what, outs=[o]), 3)
        lin["n_dirs"].append(n)
        lin["ms"].append(t)
        lin["px_per_s"].append(64 * n * T / (t * 1e-3))
        pl.close()
    lin["time_ratio_16384_vs_4096"] = lin["ms"][2] / lin["ms"][0]
    res["linearity_gpu"] = lin

    c1 = gen.config("C1")
    pc = dmas.Plan(c1["mic_xyz"], c1["dirs"], c1["fs"], c1["c"], c1["order"], c1["T"], device=dev.index,
                   max_frames=1)
    xc = torch.from_numpy(c1["signals"]).to(dev)
    oc = torch.empty((1, len(c1["dirs"]), c1["T"]), dtype=torch.float32, device=dev)
    n_rep = 100
    eager = time_fn(lambda: pc.beamform(xc, what, outs=[oc]), n_rep, warm=3)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        pc.beamform(xc, what, outs=[oc])          # warm-up on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            for _ in range(n_rep):
                pc.beamform(xc, what, outs=[oc])
    torch.cuda.synchronize()
    graph = time_fn(g.replay, 5) / n_rep
    res["latency_C1"] = {"eager_us_per_frame": 1e3 * eager, "graph_us_per_frame": 1e3 * graph,
                         "frames": n_rep, "px_per_frame": len(c1["dirs"]) * c1["T"],
                         "kernels_per_frame": 3,
                         "note": "C1: 8-mic ULA, 91 directions, T = 1024, CF-DMAS2 envelope; one dmas_beamform call "
                                 "per frame (roots, beamform, envelope); graph = 100 calls captured once, replayed"}
    pc.close()

    # the e2e's bound: device-to-host copy bandwidth into pinned memory (PCIe), 2 GiB copies
    src = flat[: (2 << 30) // 4]
    dst = torch.empty(src.numel(), dtype=torch.float32, pin_memory=True)
    d2h = time_fn(lambda: dst.copy_(src, non_blocking=True), 3)
    res["pcie_d2h_GB_s"] = src.numel() * 4 / (d2h * 1e-3) / 1e9
    return res


def main():
    args = parse()
    if args.frames <= 0:
        args.frames = WORKLOADS[args.workload]["frames"]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    # stdout carries exactly one JSON line: anything else written to fd 1 (NCCL's version banner when
    # NCCL_DEBUG=VERSION, library messages) goes to stderr; emit() writes to the saved real stdout
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.dry_run:
        return run_dry(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
