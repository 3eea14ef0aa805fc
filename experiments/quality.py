"""NEXT-4: the paper's §III-A quality sweeps driven through the GPU path.

Each sweep builds many small plans (one per array / scene), beamforms noise-free or noisy
synthetic scenes through `dmas_beamform` (matched-filtered input, 127-tap 5 kHz envelope) and
reduces the images to the paper's figures of merit:

* psf_sweep        — directional dynamic range and -3 dB range width of the PSF for DAS,
                     DMAS2..DMAS5, each without / with CF (Fig. 2);
* image_snr_sweep  — image SNR = 20 log10(1 / E_off) vs input SNR (Fig. 3);
* beamwidth_sweep  — -3 dB beamwidth vs hexagonal-array radius (Fig. 6).

Definitions the paper leaves open (reading Q20): dynamic range = peak over the largest
response more than 20 deg away from the peak direction (envelope maxima over range); the
off-target set Omega_off excludes |az - az_target| <= 15 deg and |t - t_target| <= 1125 samples
(one chirp length); beamwidth = width of the azimuth profile above -3 dB of its
peak, linearly interpolated.  The paper's absolute numbers ("almost 80 dB") depend on unstated
definitions and are not reproduced; the trends are checked (tests/test_gpu_quality.py).

    python experiments/quality.py [--out profiles/r01/quality.json]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workloads import gen  # noqa: E402

VARIANTS = [("DAS", 2, "das"), ("DMAS2", 2, "dmas"), ("DMAS3", 3, "dmas"), ("DMAS4", 4, "dmas"),
            ("DMAS5", 5, "dmas")]


def _beamform(mic, dirs, sig, p, kinds):
    """Envelope images [n_dirs][T] of `kinds` (names) for one matched-filtered frame."""
    import torch
    from paper_2511_09165_b200 import dmas
    bits = 0
    for k in kinds:
        bits |= dmas.KIND_BITS[k]
    plan = dmas.Plan(mic, dirs, gen.FS, gen.C_SOUND, p, sig.shape[-1])
    res = plan.beamform(torch.from_numpy(np.ascontiguousarray(sig[None])).cuda(), dmas.ENV(bits))
    out = {k: res[("env", k)][0].cpu().numpy().astype(np.float64) for k in kinds}
    plan.close()
    return out


def dynamic_range_db(env, az_deg, exclude_deg=20.0):
    prof = env.max(axis=1)
    a = int(np.argmax(prof))
    side = prof[np.abs(az_deg - az_deg[a]) > exclude_deg].max()
    return 20 * math.log10(prof[a] / side), a


def range_width(env, row):
    """-3 dB width (samples) of the envelope along t at the peak row."""
    r = env[row]
    t = int(np.argmax(r))
    thr = r[t] / math.sqrt(2)
    lo = t
    while lo > 0 and r[lo - 1] >= thr:
        lo -= 1
    hi = t
    while hi < len(r) - 1 and r[hi + 1] >= thr:
        hi += 1
    return hi - lo + 1


def psf_sweep(beamform=_beamform, n_mics=32):
    """Noise-free point reflector at az 10 deg, 0.5 m; 32-mic eRTIS-like array; az -90..90 step 1."""
    mic = gen.disk_array(n_mics, seed=7)
    az = np.arange(-90.0, 91.0, 1.0)
    dirs = gen.az_grid_deg(az)
    sig = gen.frame(mic, [(math.radians(10.0), 0.0, 0.5, 1.0)], 1536)
    rows = {}
    for name, p, kind in VARIANTS:
        cfk = "cfdas" if kind == "das" else "cfdmas"
        imgs = beamform(mic, dirs, sig, p, (kind, cfk))
        for cf, k in ((False, kind), (True, cfk)):
            dr, a = dynamic_range_db(imgs[k], az)
            rows[name + ("-CF" if cf else "")] = {"dynamic_range_db": dr, "peak_az_deg": float(az[a]),
                                                  "range_width_samples": range_width(imgs[k], a)}
    return rows


def image_snr(env, az_deg, az_t, t_t, guard_deg=15.0, guard_t=1125):
    img = env / env.max()
    t = np.arange(img.shape[1])
    off = (np.abs(az_deg - az_t)[:, None] > guard_deg) | (np.abs(t - t_t)[None, :] > guard_t)
    return 20 * math.log10(1.0 / img[off].mean())


def image_snr_sweep(beamform=_beamform, snrs=(-20.0, -10.0, 0.0, 10.0), seeds=(1, 2, 3)):
    """Broadside reflector at 1 m (sample 2624), unit echo amplitude, white noise of SNR_mic
    (PAPER.md:214-224); horizontal scan az -90..90 step 2, T = 4096."""
    mic = gen.disk_array(32, seed=7)
    az = np.arange(-90.0, 91.0, 2.0)
    dirs = gen.az_grid_deg(az)
    t_t = round(2 * 1.0 / gen.C_SOUND * gen.FS)
    out = {}
    for snr in snrs:
        acc = {}
        for seed in seeds:
            sig = gen.frame(mic, [(0.0, 0.0, 1.0, 1.0)], 4096, snr_db=snr, seed=seed)
            for name, p, kind in VARIANTS:
                cfk = "cfdas" if kind == "das" else "cfdmas"
                imgs = beamform(mic, dirs, sig, p, (kind, cfk))
                for cf, k in ((False, kind), (True, cfk)):
                    acc.setdefault(name + ("-CF" if cf else ""), []).append(image_snr(imgs[k], az, 0.0, t_t))
        out[str(snr)] = {k: float(np.mean(v)) for k, v in acc.items()}
    return out


def beamwidth_deg(env, az_deg):
    prof = env.max(axis=1)
    a = int(np.argmax(prof))
    thr = prof[a] / math.sqrt(2)

    def cross(step):
        i = a
        while 0 <= i + step < len(prof) and prof[i + step] >= thr:
            i += step
        j = i + step
        if not (0 <= j < len(prof)):
            return az_deg[i]
        f = (prof[i] - thr) / (prof[i] - prof[j])       # linear interpolation to the crossing
        return az_deg[i] + f * (az_deg[j] - az_deg[i])

    return abs(cross(1) - cross(-1))


def beamwidth_sweep(beamform=_beamform, radii=(0.01, 0.02, 0.04, 0.06)):
    """Hexagonal 5 mm lattice arrays, broadside reflector at 1 m, noise-free,
    az -30..30 step 0.25 deg; -3 dB width of the envelope's azimuth profile."""
    az = np.arange(-30.0, 30.01, 0.25)
    dirs = gen.az_grid_deg(az)
    out = {}
    for r in radii:
        mic = gen.hex_array(r)
        sig = gen.frame(mic, [(0.0, 0.0, 1.0, 1.0)], 3072)
        row = {"n_mics": int(len(mic))}
        for name, p, kind in VARIANTS:
            cfk = "cfdas" if kind == "das" else "cfdmas"
            imgs = beamform(mic, dirs, sig, p, (kind, cfk))
            row[name] = beamwidth_deg(imgs[kind], az)
            row[name + "-CF"] = beamwidth_deg(imgs[cfk], az)
        out[f"{r * 100:.0f}cm"] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "quality.json"))
    args = ap.parse_args()
    res = {"psf": psf_sweep(), "image_snr": image_snr_sweep(), "beamwidth": beamwidth_sweep()}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
