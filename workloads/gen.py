"""Seeded synthetic eRTIS-shaped inputs (the one module both sides may use).

Holds NONE of the beamformer's arithmetic: no delay table, no gather, no
DAS/DMAS/CF, no envelope.  It builds the *scene* (array, direction grid,
emitted chirp, analytic far-field echoes, noise, matched filter) and returns the
fp32 matched-filtered recording that the oracle and the CUDA path both consume
(SURVEY.md §8(d)).

Physical recipe (PAPER.md:253 eRTIS: 32 MEMS mics, 2.5 ms chirp 25-50 kHz,
450 kHz; PAPER.md:212 10 cm apertures; PAPER.md:214-224 noise model
m^n = m + eta n, eta = 10^(-SNR/20); PAPER.md:73 matched filter).
"""

from __future__ import annotations

import math

import numpy as np

FS = 450_000.0
C_SOUND = 343.0
CHIRP_F0, CHIRP_F1, CHIRP_DUR = 25_000.0, 50_000.0, 2.5e-3


# ------------------------------------------------------------------ arrays
def ula(n: int, spacing: float = 3.43e-3):
    """Uniform linear array on the y axis, centred at the origin (x = z = 0)."""
    y = (np.arange(n) - (n - 1) / 2.0) * spacing
    return np.stack([np.zeros(n), y, np.zeros(n)], axis=1)


def disk_array(n: int, diameter: float = 0.10, min_spacing: float = 6e-3, seed: int = 7):
    """Pseudo-random planar array: uniform in a disk in the y-z plane, rejection
    sampled with a minimum spacing, then re-centred so its centroid is the origin."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pts = []
    r = diameter / 2.0
    tries = 0
    while len(pts) < n:
        tries += 1
        if tries > 1_000_000:
            raise RuntimeError("could not place microphones")
        y, z = rng.uniform(-r, r, size=2)
        if y * y + z * z > r * r:
            continue
        if all((y - q[0]) ** 2 + (z - q[1]) ** 2 >= min_spacing ** 2 for q in pts):
            pts.append((y, z))
    yz = np.array(pts)
    yz -= yz.mean(axis=0)
    return np.stack([np.zeros(n), yz[:, 0], yz[:, 1]], axis=1)


def hex_array(radius: float, edge: float = 5e-3):
    """Microphones on a hexagonal (triangular) lattice of edge `edge`, one at the origin, all
    lattice points with |p| <= radius, in the y-z plane (Fig. 6: 5 mm edge,
    radius 1..6 cm, "19--513 microphones")."""
    n = int(radius / edge) + 2
    pts = []
    for j in range(-2 * n, 2 * n + 1):
        for i in range(-2 * n, 2 * n + 1):
            y = edge * (i + 0.5 * j)
            z = edge * (math.sqrt(3.0) / 2.0) * j
            if y * y + z * z <= radius * radius * (1 + 1e-12):
                pts.append((0.0, y, z))
    return np.array(sorted(pts, key=lambda q: (q[2], q[1])))


# ------------------------------------------------------------------ grids
def az_grid_deg(az_deg, el_deg: float = 0.0):
    az = np.deg2rad(np.asarray(az_deg, dtype=np.float64))
    return np.stack([az, np.full_like(az, math.radians(el_deg))], axis=1)


def az_el_grid(n_az: int, az_span_deg: float, n_el: int, el_span_deg: float):
    """n_az x n_el grid, linspace over +-span, elevation fastest."""
    az = np.deg2rad(np.linspace(-az_span_deg, az_span_deg, n_az))
    el = np.deg2rad(np.linspace(-el_span_deg, el_span_deg, n_el))
    A, E = np.meshgrid(az, el, indexing="ij")
    return np.stack([A.ravel(), E.ravel()], axis=1)


# ------------------------------------------------------------------ signals
def chirp_fn(t):
    """Linear FM 25 -> 50 kHz, 2.5 ms, unit amplitude, rectangular window."""
    t = np.asarray(t, dtype=np.float64)
    k = (CHIRP_F1 - CHIRP_F0) / CHIRP_DUR
    w = np.sin(2 * np.pi * (CHIRP_F0 * t + 0.5 * k * t * t))
    return np.where((t >= 0) & (t < CHIRP_DUR), w, 0.0)


def chirp_samples(fs: float = FS):
    n = int(round(CHIRP_DUR * fs))                # 1125 samples at 450 kHz
    return chirp_fn(np.arange(n) / fs)


def echoes(mic_xyz, reflectors, T_raw: int, fs: float = FS, c: float = C_SOUND):
    """Analytic far-field echoes (no interpolation): reflector (az, el, R, a) gives
    m_i(n) += a * w(n/fs - 2R/c + (p_i . u)/c) — a mic nearer the source hears it earlier."""
    mic_xyz = np.asarray(mic_xyz, dtype=np.float64)
    t = np.arange(T_raw) / fs
    out = np.zeros((mic_xyz.shape[0], T_raw))
    for (az, el, R, a) in reflectors:
        u = np.array([math.cos(el) * math.cos(az), math.cos(el) * math.sin(az), math.sin(el)])
        lead = mic_xyz @ u / c
        out += a * chirp_fn(t[None, :] - 2.0 * R / c + lead[:, None])
    return out


def matched_filter(raw, T: int, fs: float = FS):
    """Correlate each channel with the emitted chirp, / sum(w^2), keep T samples."""
    w = chirp_samples(fs)
    n = raw.shape[-1] + w.shape[0]
    nfft = 1 << (n - 1).bit_length()
    X = np.fft.rfft(raw, nfft, axis=-1)
    W = np.fft.rfft(w, nfft)
    y = np.fft.irfft(X * np.conj(W), nfft, axis=-1)[..., :T]
    return y / np.sum(w * w)


def raw_frame(mic_xyz, reflectors, T: int, snr_db=None, seed: int = 0, fs: float = FS, c: float = C_SOUND):
    """One raw (not matched-filtered) recording [n_mics][T + L], float64: echoes + noise."""
    L = int(round(CHIRP_DUR * fs))
    raw = echoes(mic_xyz, reflectors, T + L, fs, c)
    if snr_db is not None:
        eta = 10.0 ** (-snr_db / 20.0)
        rng = np.random.Generator(np.random.PCG64(seed))
        raw = raw + eta * rng.standard_normal(raw.shape)
    return raw


def frame(mic_xyz, reflectors, T: int, snr_db=None, seed: int = 0, fs: float = FS, c: float = C_SOUND):
    """One matched-filtered fp32 frame [n_mics][T]."""
    raw = raw_frame(mic_xyz, reflectors, T, snr_db, seed, fs, c)
    y = matched_filter(raw, T, fs).astype(np.float32)
    y[np.abs(y) < 1e-30] = 0.0                     # no denormal-vs-FTZ ambiguity
    return y


def random_reflectors(n: int, dirs, r_lo: float, r_hi: float, a_lo: float, a_hi: float, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    az_lo, az_hi = dirs[:, 0].min(), dirs[:, 0].max()
    el_lo, el_hi = dirs[:, 1].min(), dirs[:, 1].max()
    return [(rng.uniform(az_lo, az_hi), rng.uniform(el_lo, el_hi), rng.uniform(r_lo, r_hi),
             rng.uniform(a_lo, a_hi)) for _ in range(n)]


# ------------------------------------------------------------------ configs (BASELINE.json "configs")
def config(name: str, frames=None, stream: int = 0):
    """Scene + plan parameters of BASELINE.json configs C1..C5.

    Returns dict: mic_xyz, dirs, fs, c, order, T, signals fp32 [F][n_mics][T], plus
    metadata.  ``frames`` overrides the frame count (C5 only); ``stream`` selects an
    independent C5 frame stream (other reflectors and noise; used per rank in bench.py)."""
    if name == "C1":
        mic = ula(8)
        dirs = az_grid_deg(np.arange(-90, 91, 2))
        T, p, F = 1024, 2, 1
        refl = [(math.radians(20.0), 0.0, 600 / FS * C_SOUND / 2, 1.0)]
        sig = frame(mic, refl, T)[None]
    elif name in ("C2", "C3"):
        mic = disk_array(32, 0.10, 6e-3, seed=7)
        dirs = az_el_grid(60, 90.0, 30, 45.0)
        T, F = 4096, 1
        if name == "C2":
            p = 2
            refl = [(math.radians(10.0), math.radians(5.0), 1.0, 1.0)]
            sig = frame(mic, refl, T)[None]
        else:
            p = 5
            refl = random_reflectors(5, dirs, 0.3, 1.45, 0.2, 1.0, seed=3)
            sig = frame(mic, refl, T, snr_db=0.0, seed=3)[None]
    elif name == "C4":
        mic = disk_array(64, 0.10, 4e-3, seed=11)
        dirs = az_el_grid(128, 90.0, 128, 60.0)
        T, p = 8192, 3
        F = 1 if frames is None else int(frames)
        refl = random_reflectors(3, dirs, 0.5, 2.9, 0.3, 1.0, seed=4 + 7919 * stream)
        sig = np.empty((F, mic.shape[0], T), dtype=np.float32)
        for f in range(F):                          # frame 0 is the parity frame (noise seed 4)
            sig[f] = frame(mic, refl, T, snr_db=10.0, seed=4 + f + 1_000_003 * stream)
    elif name == "C5":
        mic = disk_array(32, 0.10, 6e-3, seed=7)
        dirs = az_el_grid(128, 90.0, 128, 60.0)
        T, p = 4096, 2
        F = 256 if frames is None else int(frames)
        base = random_reflectors(3, dirs, 0.3, 1.0, 0.3, 1.0, seed=5 + 7919 * stream)
        sig = np.empty((F, mic.shape[0], T), dtype=np.float32)
        for f in range(F):
            refl = [(az, el, R + 1e-3 * f, a) for (az, el, R, a) in base]
            sig[f] = frame(mic, refl, T, snr_db=10.0, seed=5 + f + 1_000_003 * stream)
    else:
        raise KeyError(name)
    return dict(name=name, mic_xyz=mic, dirs=dirs, fs=FS, c=C_SOUND, order=p, T=T,
                signals=np.ascontiguousarray(sig), n_frames=sig.shape[0])


def raw_config(name: str, frames=None):
    """Raw-recording variant of a config for the matched-filter path (NEXT-1): same scene, signals
    are the fp32 raw recordings [F][n_mics][T + L - 1] before pulse compression, plus the emitted
    chirp `chirp` [L] (the matched-filter template)."""
    cfg = config(name, frames=1)                 # geometry / grid / order only
    F = 1 if frames is None else int(frames)
    L = int(round(CHIRP_DUR * FS))
    mic, T = cfg["mic_xyz"], cfg["T"]
    scenes = {"C1": ([(math.radians(20.0), 0.0, 600 / FS * C_SOUND / 2, 1.0)], None),
              "C2": ([(math.radians(10.0), math.radians(5.0), 1.0, 1.0)], None),
              "C3": (random_reflectors(5, cfg["dirs"], 0.3, 1.45, 0.2, 1.0, seed=3), 0.0)}
    refl, snr = scenes.get(name, (random_reflectors(3, cfg["dirs"], 0.3, 1.0, 0.3, 1.0, seed=5), 10.0))
    sig = np.empty((F, mic.shape[0], T + L - 1), dtype=np.float32)
    for f in range(F):
        sig[f] = raw_frame(mic, refl, T, snr_db=snr, seed=3 + f)[:, :T + L - 1].astype(np.float32)
    cfg.update(signals=np.ascontiguousarray(sig), n_frames=F, chirp=chirp_samples(FS).astype(np.float32))
    return cfg


def random_signals(F: int, n_mics: int, T: int, seed: int, scale: float = 1.0, sparsity: float = 0.0):
    """Plain Gaussian test signals (edge cases / stress), fp32, optional exact zeros."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = (scale * rng.standard_normal((F, n_mics, T))).astype(np.float32)
    if sparsity > 0:
        x[rng.random(x.shape) < sparsity] = 0.0
    x[np.abs(x) < 1e-30] = 0.0
    return x
