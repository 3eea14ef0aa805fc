"""The paper's execution-time workload (Table I / Table II) on one B200, as
context next to the paper's own numbers (their hardware).

Workload: a 32-microphone eRTIS recording, 1000 directions, one frame; the
sample count is printed inconsistently ("163 840 samples (0.0364 s at 450 kHz)"), so both
readings are timed: T = 16,384 and T = 163,840.  Directions: 1000 azimuths over -90..90 deg at
elevation 0 (the paper's Fig. 7 sweeps azimuth counts).  Methods: DAS, DMAS2..5 and DMAS2-CF,
raw beamformer output (the paper times its beamforming kernel).  Device time per frame with CUDA
events around dmas_beamform, median of 50 frames after 5 warm-ups ("executed 50
times"); the root prologue is included.

usage: python tools/paper_table.py [--out profiles/r01/paper_table.json]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_09165_b200 import dmas  # noqa: E402
from workloads import gen  # noqa: E402

# PAPER.md:273-279 (Table I, ms) and :294-300 (Table II, DMAS2-CF ms), RTX 3090 and Orin AGX rows
PAPER_MS = {"RTX 3090": {"DAS": 20, "DMAS2": 21, "DMAS3": 26, "DMAS4": 32, "DMAS5": 40, "DMAS2-CF": 21},
            "Jetson Orin AGX": {"DAS": 20, "DMAS2": 37, "DMAS3": 79, "DMAS4": 129, "DMAS5": 184, "DMAS2-CF": 38}}


def time_method(mic, dirs, T, p, kind, reps=50, warm=5):
    plan = dmas.Plan(mic, dirs, gen.FS, gen.C_SOUND, p, T, max_frames=1, lp_taps=0)
    rng = np.random.default_rng(T + p)
    x = torch.from_numpy(rng.standard_normal((1, mic.shape[0], T)).astype(np.float32)).cuda()
    out = [torch.empty((1, len(dirs), T), device="cuda")]
    st = torch.cuda.current_stream()
    times = []
    for r in range(warm + reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        plan.beamform(x, dmas.RAW(kind), outs=out)
        e1.record(st)
        e1.synchronize()
        if r >= warm:
            times.append(e0.elapsed_time(e1))
    info = plan.info
    plan.close()
    return statistics.median(times), info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    mic = gen.disk_array(32, 0.10, 6e-3, seed=7)
    dirs = gen.az_grid_deg(np.linspace(-90.0, 90.0, 1000))
    methods = [("DAS", 2, dmas.KIND_DAS), ("DMAS2", 2, dmas.KIND_DMAS), ("DMAS3", 3, dmas.KIND_DMAS),
               ("DMAS4", 4, dmas.KIND_DMAS), ("DMAS5", 5, dmas.KIND_DMAS), ("DMAS2-CF", 2, dmas.KIND_CFDMAS)]
    rows = []
    for T in (16384, 163840):
        for name, p, kind in methods:
            ms, info = time_method(mic, dirs, T, p, kind)
            row = {"T": T, "method": name, "b200_ms_per_frame": ms, "b200_Gpx_s": 1000 * T / (ms * 1e-3) / 1e9,
                   "bf_kernel": info["bf_kernel"]}
            for gpu, tab in PAPER_MS.items():
                row[f"paper_{gpu}_ms"] = tab[name]
                row[f"speedup_vs_{gpu}"] = tab[name] / ms
            rows.append(row)
            print(f"T {T:6d} {name:9s} B200 {ms:8.4f} ms/frame ({row['b200_Gpx_s']:6.1f} Gpx/s)   "
                  f"paper RTX 3090 {PAPER_MS['RTX 3090'][name]:4d} ms   Orin AGX {PAPER_MS['Jetson Orin AGX'][name]:4d} ms",
                  flush=True)
    doc = {"workload": "PAPER.md:264 - 32 mics (eRTIS-like disk), 1000 azimuths (-90..90 deg, el 0), one frame, "
                       "raw beamformer output; T = 16384 and 163840 (the paper's two readings)",
           "timing": "CUDA events around dmas_beamform (roots prologue + beamform), median of 50 after 5 warm-ups",
           "paper_source": "PAPER.md:273-279 (Table I), :294-300 (Table II); their hardware, context only",
           "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
