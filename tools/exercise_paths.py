"""Run every kernel path once on small inputs (for compute-sanitizer / quick checks on a GPU box):
nearest and linear pre-steering, orders 2..8, tensor-core / FP32 / generic envelopes, band-pass,
decimation, matched filter, host pipeline, ragged shapes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_09165_b200 import dmas  # noqa: E402
from workloads import gen  # noqa: E402


def main():
    allk = dmas.RAW(dmas.KIND_ALL) | dmas.ENV(dmas.KIND_ALL)
    mic = gen.disk_array(16, seed=5)
    dirs = gen.az_el_grid(9, 60.0, 5, 30.0)
    for T in (4096 + 32, 700, 33):
        sig = torch.from_numpy(gen.random_signals(2, 16, T, seed=T)).cuda()
        for p in (2, 3, 5, 8):
            for kw in ({}, {"delay_interp": 1}, {"env_engine": 1}, {"env_decim": 3, "lp_taps": 63},
                       {"bp_coeffs": np.hanning(15)}):
                plan = dmas.Plan(mic, dirs, gen.FS, gen.C_SOUND, p, T, max_frames=2, **kw)
                plan.beamform(sig, allk)
                plan.beamform(sig, dmas.ENV(dmas.KIND_CFDMAS))
                plan.close()
    cfg = gen.raw_config("C1", frames=2)
    plan = dmas.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=1,
                     mf_coeffs=cfg["chirp"])
    plan.beamform_host(cfg["signals"], allk)
    torch.cuda.synchronize()
    print("exercise_paths OK, kernels launched:", dmas.launch_count())


if __name__ == "__main__":
    main()
