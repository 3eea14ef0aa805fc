#!/usr/bin/env python
"""Throughput benchmark of the DMAS / CF beamforming hot path on B200.

Metric (BASELINE.json): "CF-DMAS images/sec (directions x range samples per second)", i.e.
pixels/s = frames * n_dirs * T / time.  Workload: BASELINE.json configs[4] = C5, the streaming
config the metric's 1/2/4/8-GPU throughput is quoted on: 32-mic eRTIS-like
array, 16,384 directions (128 az x 128 el), T = 4096 at 450 kHz, 256 frames per step, CF-DMAS
p = 2 followed by the 127-tap 5 kHz envelope.  One step = one dmas_beamform call over the
256-frame batch (every §8(a) row: signed roots -> gather / power sums / Newton-Girard / CF ->
envelope); the delay table (A1) is built once per plan, as the paper pre-computes it.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path (one process per GPU)
  python bench.py --impl reference ...                      # the float64 oracle on the host cores

Multi-GPU (torchrun, one rank per GPU, NCCL): frames are independent problems, so every rank
beamforms its own 256-frame stream over the full grid (weak scaling, no data-path collective);
the step time is the max over ranks.  ``--mode dirshard`` instead broadcasts one stream from
rank 0 and splits the direction grid (strong scaling; shards stay resident).
"""

from __future__ import annotations

import argparse
import json
import os
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
FP32_LANES_PER_SM_CLK = 128     # FFMA/FADD/FMUL lanes per SM per clock (B200, measured 124-128)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=0, help="frames per step (0: the workload's, C5 256, C4 16)")
    ap.add_argument("--workload", choices=["C5", "C4"], default="C5",
                    help="C5 = the metric's config (default); C4 = 64-mic p = 3 secondary line")
    ap.add_argument("--mode", choices=["weak", "dirshard"], default="weak")
    ap.add_argument("--bf-engine", type=int, choices=[0, 1], default=0,
                    help="beamform kernel: 0 auto (LDS.64 kernel where it fits), 1 classic k_beamform (comparison)")
    ap.add_argument("--interp", action="store_true",
                    help="linear-interpolation pre-steering (fractional delays, roots on the fly; NEXT-2)")
    ap.add_argument("--raw", action="store_true",
                    help="raw recordings in: the step includes the GPU matched filter (paper Fig. 1 pipeline)")
    ap.add_argument("--e2e-frames", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-dirs", type=int, default=0, help="directions per core in the CPU sample (0 = auto)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def _oracle_chunk(job):
    from oracle import dmas_oracle as O
    sig, d, p = job
    h = O.lpf_taps(LP_TAPS, 5000.0, gen.FS)
    img = O.beamform_frame(sig, d, p)
    e = O.envelope(img["cfdmas"], h)
    return e.shape[0] * e.shape[1]


def oracle_rate(cfg, frame_idx=0, dirs_per_core=0, cores=None, pool=None):
    """Time the float64 oracle (as it stands) on a bounded sample of the C5 step: one frame,
    `cores` x `dirs_per_core` directions (default: the whole frame), all T samples, CF-DMAS +
    envelope, one process per core over contiguous direction chunks.  The delay table is built
    outside the timed region, as in the CUDA path's plan.  Returns (px/s, cores, description)."""
    import multiprocessing as mp
    from oracle import dmas_oracle as O
    cores = cores or os.cpu_count() or 1
    dpc = dirs_per_core or max(1, -(-len(cfg["dirs"]) // cores))    # default: one whole frame
    n = min(len(cfg["dirs"]), cores * dpc)
    sel = np.linspace(0, len(cfg["dirs"]) - 1, n).astype(int)
    d = O.delay_table(cfg["mic_xyz"], cfg["dirs"][sel], cfg["fs"], cfg["c"])
    jobs = [(cfg["signals"][frame_idx], d[i:i + dpc], cfg["order"]) for i in range(0, n, dpc)]
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
    desc = (f"frame {frame_idx} of {cfg['name']}, {n} of {len(cfg['dirs'])} directions x {cfg['T']} samples "
            f"= {px} px, CF-DMAS p={cfg['order']} + {LP_TAPS}-tap envelope, float64 numpy oracle, "
            f"{cores} processes; {dt:.1f} s")
    return px / dt, cores, desc


def run_reference(args, rank, world):
    """The reference arm: the oracle, as it stands, on the host cores (rank 0 only).  Each step
    beamforms one whole C5 frame (a bounded sample of the 256-frame step) with a process pool
    over all cores; value = median px/s over the timed steps."""
    import multiprocessing as mp
    if rank != 0:
        return 0
    cfg = gen.config(args.workload, frames=1)
    cores = os.cpu_count() or 1
    rates, desc = [], ""
    with mp.get_context("fork").Pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            r, c, desc = oracle_rate(cfg, 0, args.cpu_dirs, cores, pool)
            if i >= args.warmup:
                rates.append(r)
    value = statistics.median(rates)
    px_step = len(cfg["dirs"]) * cfg["T"] * args.frames
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * px_step / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "each step times one whole C5 frame (a bounded sample of the 256-frame step) on the host cores; "
                "ms_per_step is that rate extrapolated linearly to the 256-frame step (cost is exactly "
                "proportional to frames x directions x samples)",
    }
    print(json.dumps(line), flush=True)
    return 0


def load_traffic():
    """DRAM bytes per launch of each kernel from the committed `ncu --set full` capture
    (profiles/<round>/traffic.json, written from dram__bytes_read.sum + dram__bytes_write.sum)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
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
# FP32-pipe lane-ops per microphone sample of k_beamform (acc_add<P>) and per pixel
# epilogue (Newton-Girard + CF + CF product)
OPS_PER_MIC = {2: 5, 3: 6, 4: 10, 5: 10}
BF_KERNELS = {0: "k_beamform", 1: "k_beamform_lds64", 2: "k_beamform_mg"}   # dmas_plan_info.bf_kernel
OPS_EPI = {2: 6, 3: 10, 4: 14, 5: 18}


def config_dict(args, world):
    w = WORKLOADS[args.workload]
    return {"workload": args.workload, "array": w["array"], "n_dirs": w["n_dirs"], "grid": w["grid"],
            "n_samples": w["n_samples"], "fs_hz": w["fs_hz"], "order": w["order"],
            "frames_per_step_per_gpu": args.frames,
            "outputs": f"CF-DMAS{w['order']} envelope (127-tap 5 kHz low-pass)",
            "mode": args.mode, "world": world, "l2": w["l2"],
            "input": "raw recordings, matched filter on the GPU (1125-tap chirp)" if args.raw
                     else "matched-filtered signals (north_star input)",
            "presteer": "linear interpolation (fractional delays)" if args.interp else "nearest sample (integer LUT)",
            "beamform_kernel": "classic k_beamform (forced)" if args.bf_engine == 1 else "auto"}


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


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local):
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_cfg = gen.config(args.workload, frames=1)
        r, c, desc = oracle_rate(cpu_cfg, 0, args.cpu_dirs, None)
        cpu = {"value": r, "unit": UNIT, "cores": c, "kind": "oracle", "sample": desc}

    import torch
    import torch.distributed as dist
    from paper_2511_09165_b200 import dmas, parallel

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- inputs (resident in HBM before the timed region)
    if args.raw:
        cfg = gen.raw_config(args.workload, frames=args.frames)
        dirs = cfg["dirs"]
        x = torch.from_numpy(cfg["signals"]).to(dev)
    elif args.mode == "weak":
        cfg = gen.config(args.workload, frames=args.frames, stream=rank)
        dirs = cfg["dirs"]
        x = torch.from_numpy(cfg["signals"]).to(dev)
    else:
        cfg = (gen.config(args.workload, frames=args.frames, stream=0) if rank == 0
               else gen.config(args.workload, frames=1))
        g0, g1 = parallel.partition(len(cfg["dirs"]), world, rank)
        dirs = cfg["dirs"][g0:g1]
        x = torch.empty((args.frames, cfg["mic_xyz"].shape[0], cfg["T"]), dtype=torch.float32, device=dev)
        if rank == 0:
            x.copy_(torch.from_numpy(cfg["signals"]))
    F, T, p = args.frames, cfg["T"], cfg["order"]
    plan = dmas.Plan(cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], p, T, max_frames=F, lp_taps=LP_TAPS, device=local,
                     mf_coeffs=cfg.get("chirp") if args.raw else None, delay_interp=1 if args.interp else 0, bf_engine=args.bf_engine)
    bf_name = BF_KERNELS[plan.info["bf_kernel"]]
    what = dmas.ENV(dmas.KIND_CFDMAS)
    out = torch.empty((F, len(dirs), T), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        if args.mode == "dirshard" and world > 1:
            dist.broadcast(x, src=0)          # signals broadcast once per step over NVLink (NCCL)
        plan.beamform(x, what, outs=[out])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(physical_gpu_index(local))
    time.sleep(0.3)
    plan.set_timing(True)
    n_launch0 = dmas.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = dmas.launch_count() - n_launch0
    plan.set_timing(False)
    ktime = plan.timing_read()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        if dist.get_rank() == 0 and clk is not None:
            pass
    n_dirs_total = len(cfg["dirs"]) if args.mode == "dirshard" else len(cfg["dirs"]) * world
    px_step = F * n_dirs_total * T
    value = px_step / (ms * 1e-3)

    # ---- roofline of the dominant kernel (device time inside the timed region)
    bf_ms, bf_n = ktime["beamform"]
    env_ms, env_n = ktime["envelope"]
    rt_ms, rt_n = ktime["signed_roots"]
    px_launch_bf = (F * len(dirs) * T) / max(1, bf_n / args.steps)   # pixels per beamform launch
    n_mics = cfg["mic_xyz"].shape[0]
    ops_bf = OPS_PER_MIC[p] * n_mics + OPS_EPI[p]   # FP32 pipe lane-ops per pixel
    ops_env = LP_TAPS                            # one FFMA per tap per pixel
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = (clk or {}).get("sm_max_mhz") or 1965.0
    peak_top = FP32_LANES_PER_SM_CLK * sm_count * sm_max * 1e6 / 1e12     # T lane-ops/s at max clock
    bf_avg = bf_ms / max(1, bf_n)
    env_avg = env_ms / max(1, env_n)
    px_launch_env = (F * len(dirs) * T) / max(1, env_n / args.steps)
    ach_bf = ops_bf * px_launch_bf / (bf_avg * 1e-3) / 1e12
    ach_env = ops_env * px_launch_env / (env_avg * 1e-3) / 1e12
    hbm_peak = 6547.2
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    env_gbs = 8.0 * px_launch_env / (env_avg * 1e-3) / 1e9          # read raw + write envelope, 4 B each
    traffic = load_traffic()
    dom = "beamform" if bf_ms >= env_ms else "envelope"
    tr = traffic.get(f"k_{dom}", {})
    frames_launch = F / max(1, bf_n / args.steps)
    traffic_launch = (tr["dram_bytes_per_launch"] * frames_launch / tr["frames_per_launch"]
                      if tr.get("dram_bytes_per_launch") and tr.get("frames_per_launch") else None)
    if dom == "beamform":
        roofline = {"bound": "alu", "kernel": bf_name, "achieved": ach_bf, "peak": peak_top,
                    "unit": "Top/s (FP32 lane-ops)", "frac": ach_bf / peak_top}
    else:
        roofline = {"bound": "hbm", "kernel": "k_envelope_tc", "achieved": env_gbs, "peak": hbm_peak, "unit": "GB/s",
                    "frac": env_gbs / hbm_peak}
    roofline.update({"traffic": traffic_launch,
                     "traffic_unit": "bytes per launch (ncu dram read+write, scaled to this launch's frames)",
                     "algorithmic_bytes": 4.0 * px_launch_bf if dom == "beamform" else 8.0 * px_launch_env,
                "peak_basis": (f"{FP32_LANES_PER_SM_CLK} FP32 lanes/clk/SM x {sm_count} SMs x {sm_max:.0f} MHz "
                               "(guide unit counts; measured 124/128 in round-1 microbenchmark)") if dom == "beamform"
                              else "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                "kernels": {
                    "beamform": {"avg_ms": bf_avg, "launches": bf_n, "share": bf_ms / (ms * args.steps),
                                 "ops_per_px": ops_bf, "Top_s": ach_bf, "frac": ach_bf / peak_top,
                                 "Gpx_s": px_launch_bf / (bf_avg * 1e-3) / 1e9},
                    "envelope": {"avg_ms": env_avg, "launches": env_n, "share": env_ms / (ms * args.steps),
                                 "bound": "hbm", "GB_s": env_gbs, "hbm_frac": env_gbs / hbm_peak,
                                 "algorithmic_bytes_per_px": 8, "Gpx_s": px_launch_env / (env_avg * 1e-3) / 1e9},
                    "signed_roots": {"avg_ms": rt_ms / max(1, rt_n), "launches": rt_n,
                                     "share": rt_ms / (ms * args.steps)}}})

    # ---- end to end through the public API with host buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e and args.mode == "weak" and not args.raw:
        Fe = min(args.e2e_frames, F)
        hsig = torch.from_numpy(cfg["signals"][:Fe]).pin_memory()
        hout = torch.empty((Fe, len(dirs), T), dtype=torch.float32).pin_memory()
        sig_np = hsig.numpy()
        plan.beamform_host(sig_np, what, outs=[hout.numpy()])           # warm-up (allocates staging)
        if world > 1:
            dist.barrier()
        times = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            plan.beamform_host(sig_np, what, outs=[hout.numpy()])
            times.append(time.perf_counter() - t0)
        et = statistics.median(times)
        if world > 1:
            t = torch.tensor([et], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": Fe * len(dirs) * T * world / et, "unit": UNIT,
               "h2d_bytes_per_step": int(hsig.numel() * 4), "d2h_bytes_per_step": int(hout.numel() * 4),
               "frames_per_step": Fe, "timing": "host wall clock around the synchronous dmas_beamform_host call "
                                                "(pinned host buffers; H2D, kernels and D2H pipelined in chunks)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.mode == "weak" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded eRTIS-like point-reflector echoes, matched-filtered; workloads/gen.py)",
            "config": dict(config_dict(args, world), beamform_kernel=bf_name), "frames_per_s": F * (world if args.mode == "weak" else 1) / (ms * 1e-3),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.frames <= 0:
        args.frames = WORKLOADS[args.workload]["frames"]
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
