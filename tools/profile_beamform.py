"""Small driver for ncu captures of the beamform / envelope kernels: one C5-shaped plan
(32 mics, 16384 directions, T = 4096, CF-DMAS2 envelope), `--frames` frames per call,
`--calls` calls.  Usage (on a GPU box):
    python tools/profile_beamform.py --frames 8 --calls 3 [--workload C4] [--raw]
    ncu --set full -k regex:k_beamform -s 1 -c 1 -o gpurun_out/bf python tools/profile_beamform.py ...
DMAS_LIBRARY=<path to a variant libdmas.so> compares builds (dmas.py honours it).
Prints the per-kernel device time of the last call (CUDA events inside the library)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_09165_b200 import dmas  # noqa: E402
from workloads import gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--engine", type=int, default=0, help="bf_engine: 0 auto, 1 classic")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--raw", action="store_true", help="raw CF-DMAS output instead of the envelope")
    ap.add_argument("--order", type=int, default=0, help="override the workload's DMAS order")
    ap.add_argument("--env-engine", type=int, default=0, help="env_engine: 0 auto, 1 FP32 FIR, 2 tcgen05 on fp32")
    args = ap.parse_args()
    cfg = gen.config(args.workload, frames=min(args.frames, 4))
    sig = torch.from_numpy(cfg["signals"]).cuda()
    sig = sig.repeat((args.frames + sig.shape[0] - 1) // sig.shape[0], 1, 1)[:args.frames].contiguous()
    plan = dmas.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], args.order or cfg["order"], cfg["T"],
                     max_frames=args.frames, bf_engine=args.engine, env_engine=args.env_engine)
    what = dmas.RAW(dmas.KIND_CFDMAS) if args.raw else dmas.ENV(dmas.KIND_CFDMAS)
    outs = None
    for c in range(args.calls):
        plan.set_timing(c == args.calls - 1)
        res = plan.beamform(sig, what, outs)
        outs = list(res.values())
    torch.cuda.synchronize()
    t = plan.timing_read()
    px = args.frames * len(cfg["dirs"]) * cfg["T"]
    print({"info": plan.info, "timing_ms": t,
           "beamform_Gpx_s": px / (t["beamform"][0] * 1e-3) / 1e9 if t["beamform"][1] else None})


if __name__ == "__main__":
    main()
