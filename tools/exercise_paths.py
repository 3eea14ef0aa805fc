"""Run every kernel path once on small inputs (for compute-sanitizer / quick checks on a GPU box):
nearest and linear pre-steering, orders 2..8, tensor-core / FP32 / generic envelopes, band-pass,
decimation, matched filter, host pipeline, ragged shapes, every beamform kernel (classic, LDS.64
with consecutive / k-d tiles and 8 / 4 pixels per lane, microphone groups)."""
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
    # classic kernel (forced), LDS.64 k-d tiles (an elevation-fastest grid whose columns straddle
    # tiles) and LDS.64 with 4 pixels per lane (64 microphones), large-array microphone groups
    for mic_n, grid, kw in ((16, gen.az_el_grid(9, 60.0, 5, 30.0), {"bf_engine": 1}),
                            (32, gen.az_el_grid(12, 90.0, 30, 45.0), {}),
                            (64, gen.az_el_grid(8, 90.0, 40, 60.0), {}),
                            (160, gen.az_el_grid(5, 60.0, 3, 20.0), {})):
        m = gen.disk_array(mic_n, 0.10, 4e-3 if mic_n <= 64 else 3.5e-3, seed=mic_n)
        for T in (1024 + 96, 301):
            sig = torch.from_numpy(gen.random_signals(1, mic_n, T, seed=T + mic_n)).cuda()
            for p in (2, 3):
                plan = dmas.Plan(m, grid, gen.FS, gen.C_SOUND, p, T, max_frames=1, **kw)
                plan.beamform(sig, allk)
                print(f"  mics {mic_n} T {T} p {p}: bf_kernel {plan.info['bf_kernel']} tile_order "
                      f"{plan.info['tile_order']} t_tile {plan.info['t_tile']}")
                plan.close()
    cfg = gen.raw_config("C1", frames=2)
    plan = dmas.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=1,
                     mf_coeffs=cfg["chirp"])
    plan.beamform_host(cfg["signals"], allk)
    torch.cuda.synchronize()
    print("exercise_paths OK, kernels launched:", dmas.launch_count())


if __name__ == "__main__":
    main()
