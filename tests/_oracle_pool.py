"""Whole-frame oracle comparisons at full size, in a process pool (test infrastructure).

The float64 oracle needs ~70 s of one core per C5 frame, so full frames are split into
direction chunks (rows are independent: every pixel's DAS / DMAS / CF depends only on its
own (psi, t), and the envelope runs along t within one row) and farmed out
to all host cores.  Each worker beamforms its chunk with the oracle and returns, per
(stage, kind), the largest |gpu - oracle| and the largest |oracle| of the chunk; the caller
takes maxima over chunks, so the bar max|gpu - oracle| <= 1e-4 * max|oracle| is checked over
the WHOLE frame exactly as for the small configs.  The GPU images reach the workers through
fork (copy-on-write globals); the workers never touch CUDA.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from oracle import dmas_oracle as O

_G = {}


def _work(job):
    f, a0, a1 = job
    g = _G
    d = g["d"][a0:a1]
    img = O.beamform_frame(g["signals"][f], d, g["p"], eps=g["eps"], chunk=16)
    out = {}
    for (stage, kind), arr in g["gpu"].items():
        ref = img[kind] if stage == "raw" else O.envelope(img[kind], g["h"])
        got = arr[g["frame_pos"][f]][a0:a1].astype(np.float64)
        out[(stage, kind)] = (float(np.max(np.abs(got - ref))), float(np.max(np.abs(ref))),
                              bool(np.all(np.isfinite(got))))
    return f, out


def compare_frames(signals, d, p, gpu, frames, *, h=None, eps=1e-30, chunk=256, cores=None):
    """gpu: {(stage, kind): ndarray [len(frames)][n_dirs][T']} (host copies of the CUDA images for
    `frames`, in that order); signals [F][n_mics][T]; d = the oracle delay table.  Returns
    {(stage, kind, frame): (max_err, peak, finite)} over the whole frame."""
    n_dirs = d.shape[0]
    _G.clear()
    _G.update(signals=signals, d=d, p=p, eps=eps, h=h if h is not None else O.lpf_taps(), gpu=gpu,
              frame_pos={f: i for i, f in enumerate(frames)})
    jobs = [(f, a0, min(n_dirs, a0 + chunk)) for f in frames for a0 in range(0, n_dirs, chunk)]
    res = {}
    with mp.get_context("fork").Pool(cores or os.cpu_count() or 1) as pool:
        for f, out in pool.imap_unordered(_work, jobs):
            for (stage, kind), (err, peak, fin) in out.items():
                e0, p0, f0 = res.get((stage, kind, f), (0.0, 0.0, True))
                res[(stage, kind, f)] = (max(e0, err), max(p0, peak), f0 and fin)
    _G.clear()
    return res
