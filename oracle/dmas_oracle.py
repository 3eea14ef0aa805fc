"""Plain, slow, float64 oracle of the DMAS / CF beamforming hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Written from the paper
(arXiv 2511.09165, ``/root/reference/PAPER.md``; citations are ``PAPER.md:<line>``)
in the paper's order and notation.  Nothing here is blocked, fused or reordered
beyond what the cited definition states.  Readings of silent/ambiguous points
are the ones in DESIGN.md "Readings" (Q1..Q18, numbering of SURVEY.md §8(c)).

Notation (Q1): the paper's N (microphones) is ``n_mics`` / N_m, the
paper's M (directions) is ``n_dirs`` / N_psi, the DMAS order n is ``p``.

Functions are written so that the scalar-level ones (``esp_vieta``,
``brute_force_esp``, ``newton_girard_*``, ``dmas_pairwise_eq3``) accept any
number type, including ``fractions.Fraction``, so the tests can check identities
exactly.
"""

from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

# Output image kinds, in the bit order of the C ABI's output mask.
KIND_NAMES = ("das", "dmas", "cfdmas", "cfdas", "cf")


# --------------------------------------------------------------------------------------
# A1  Delay look-up table   (Sec. II; Eq. (1))
# --------------------------------------------------------------------------------------
def unit_vector(az: float, el: float):
    """Unit vector of direction psi = (theta, phi) = (azimuth, elevation).

    PAPER.md:77: "directions are defined by their azimuth and elevation angles
    (theta, phi)".  Frame (reading Q3): x = broadside, theta from +x toward +y,
    phi toward +z.  Uses Python ``math`` (glibc libm), never numpy's vectorised
    sin/cos (reading Q4: the table must be bit-exact).
    """
    ce = math.cos(el)
    return (ce * math.cos(az), ce * math.sin(az), math.sin(el))


def delay_table(mic_xyz, dir_az_el, fs: float, c: float, reference=None, return_exact=False, mode="nearest"):
    """Integer-sample delay LUT d[psi][i] ("pre-computed and stored in
    a delay matrix look-up table").

    tau_{i,psi} = -((p_i - r) . u(psi)) / c   (reading Q2: a microphone nearer
    the source hears the wave earlier, so Eq. (1) m_i(t + tau) aligns it), in
    samples v = tau * fs, rounded to the nearest sample with ties to even
    (reading Q4; Python ``round`` is ties-to-even).  Operation order, fixed for
    bit-exactness (CPython never contracts into FMA):

        dot = ((px - rx)*ux + (py - ry)*uy) + (pz - rz)*uz
        v   = dot * k,   k = -(fs / c)

    Returns int32 [n_dirs][n_mics] (and the exact float v if ``return_exact``).
    ``mode="linear"`` (NEXT-2, reading Q4b): returns (d0, alpha) with d0 = floor(v) (int32) and
    alpha = v - d0 in [0, 1) (float64) for linear-interpolation pre-steering.
    """
    mic_xyz = np.asarray(mic_xyz, dtype=np.float64)
    dir_az_el = np.asarray(dir_az_el, dtype=np.float64)
    if c <= 0 or fs <= 0:
        raise ValueError("c and fs must be positive")
    if mic_xyz.shape[0] < 1 or dir_az_el.shape[0] < 1:
        raise ValueError("empty array or grid")
    rx, ry, rz = (0.0, 0.0, 0.0) if reference is None else (float(v) for v in reference)
    k = -(float(fs) / float(c))
    n_dirs, n_mics = dir_az_el.shape[0], mic_xyz.shape[0]
    d = np.empty((n_dirs, n_mics), dtype=np.int32)
    v_exact = np.empty((n_dirs, n_mics), dtype=np.float64) if (return_exact or mode == "linear") else None
    mics = [tuple(float(q) for q in row) for row in mic_xyz]
    for a in range(n_dirs):
        ux, uy, uz = unit_vector(float(dir_az_el[a, 0]), float(dir_az_el[a, 1]))
        for i, (px, py, pz) in enumerate(mics):
            dot = ((px - rx) * ux + (py - ry) * uy) + (pz - rz) * uz
            v = dot * k
            d[a, i] = round(v) if mode == "nearest" else math.floor(v)
            if return_exact or mode == "linear":
                v_exact[a, i] = v
    if mode == "linear":
        return d, v_exact - d
    return (d, v_exact) if return_exact else d


# --------------------------------------------------------------------------------------
# A0  Matched filter (pulse compression)   (step 1 of the pipeline; NEXT-1)
# --------------------------------------------------------------------------------------
def matched_filter(raw, w, T: int):
    """m_i(t) = sum_k w[k] raw_i[t + k] / sum_k w[k]^2  for t in [0, T)   ("convolved
    with the known emitted source signal" = correlation with the emitted chirp w; reading Q19:
    normalised by the chirp energy so an exact unit echo peaks at 1, output sample t = echo onset
    t, input length T + L - 1).  Direct form, float64.  ``raw``: [..., >= T + L - 1]."""
    raw = np.asarray(raw, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    L = w.shape[0]
    if raw.shape[-1] < T + L - 1:
        raise ValueError("raw recording shorter than T + L - 1")
    out = np.zeros(raw.shape[:-1] + (T,), dtype=np.float64)
    for k in range(L):
        out += w[k] * raw[..., k:k + T]
    return out / np.sum(w * w)


# --------------------------------------------------------------------------------------
# A2  Pre-steering / delay-and-gather   (Eq. (1))
# --------------------------------------------------------------------------------------
def gather(m, d):
    """x_i(t, psi) = m_i(t + tau_{i,psi})  (Eq. (1)).

    ``m``: [n_mics][T] samples (promoted to float64); ``d``: int [n_dirs][n_mics].
    Reads outside [0, T) are 0 (reading Q5).  Returns float64 [n_dirs][n_mics][T].
    """
    m = np.asarray(m, dtype=np.float64)
    d = np.asarray(d, dtype=np.int64)
    n_mics, T = m.shape
    x = np.zeros((d.shape[0], n_mics, T), dtype=np.float64)
    for a in range(d.shape[0]):
        for i in range(n_mics):
            s = int(d[a, i])
            lo, hi = max(0, -s), min(T, T - s)  # t range with 0 <= t + s < T
            if lo < hi:
                x[a, i, lo:hi] = m[i, lo + s:hi + s]
    return x


def gather_linear(m, d0, alpha):
    """Fractional-delay pre-steering by linear interpolation (Eq. (1) PAPER.md:79 with a
    non-integer delay; reading Q4b, "fractional-sample interpolation"):
    x_i(t, psi) = (1 - a) m_i[t + d0] + a m_i[t + d0 + 1], a = alpha[psi][i]; samples outside
    [0, T) are 0.  Returns float64 [n_dirs][n_mics][T]."""
    m = np.asarray(m, dtype=np.float64)
    lo = gather(m, d0)
    hi = gather(m, np.asarray(d0, dtype=np.int64) + 1)
    a = np.asarray(alpha, dtype=np.float64)[:, :, None]
    return (1.0 - a) * lo + a * hi


# --------------------------------------------------------------------------------------
# A3  Signed roots and power sums   (Eq. power sums PAPER.md:129-133)
# --------------------------------------------------------------------------------------
def signed_root(x, p: int):
    """s_i^(n) = sgn(x_i) * |x_i|^(1/n).  sgn(0) = 0 (reading Q6)."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.power(np.abs(x), 1.0 / p)


def power_sums(s, p: int, axis: int = 0):
    """P_k^(n) = sum_i (s_i^(n))^k for k = 1..n   (Eq. PAPER.md:131).  Returns [P_1..P_p]."""
    s = np.asarray(s, dtype=np.float64)
    return [np.sum(s ** k, axis=axis) for k in range(1, p + 1)]


# --------------------------------------------------------------------------------------
# Elementary symmetric polynomial E_n  (Eq. (5), Eq. (6))
# --------------------------------------------------------------------------------------
def esp_vieta(s_list, p: int):
    """E_p(s_1..s_N) by the Vieta recurrence of prod_i (1 + s_i z) = sum_k E_k z^k.

    S_DMAS^(n) = E_n(s_1..s_N)  (Eq. (6)).  e_0 = 1; for each
    microphone i, for k = p..1: e_k += s_i * e_{k-1}.  Exact identity, O(N p),
    algorithmically disjoint from the Newton-Girard route the GPU takes.
    ``s_list`` iterates over microphones; elements may be scalars (any number
    type, e.g. Fraction) or equally shaped numpy arrays (vectorised over pixels).
    """
    e = [1] + [0] * p
    for si in s_list:
        for k in range(p, 0, -1):
            e[k] = e[k] + si * e[k - 1]
    return e[p]


def brute_force_esp(s_list, p: int):
    """Eq. (5) literally: sum over all n-subsets of the product of
    signed roots.  O(N^p): tiny inputs only (guard C(N,p) <= 1e6)."""
    s_list = list(s_list)
    if math.comb(len(s_list), p) > 10 ** 6:
        raise ValueError("brute force refused: C(N,p) too large")
    total = 0
    for comb in itertools.combinations(s_list, p):
        prod = 1
        for v in comb:
            prod = prod * v
        total = total + prod
    return total


def dmas_pairwise_eq3(x_list):
    """Eq. (3) literally: sum_{i<j} sgn(x_i x_j) sqrt(|x_i x_j|)."""
    x_list = [float(v) for v in x_list]
    total = 0.0
    n = len(x_list)
    for i in range(n - 1):
        for j in range(i + 1, n):
            q = x_list[i] * x_list[j]
            total += math.copysign(math.sqrt(abs(q)), q) if q != 0 else 0.0
    return total


def newton_girard_explicit(P, n: int):
    """The paper's pre-expanded Newton-Girard formulas for n = 2..5
    (Eqs.).  ``P[k-1]`` = P_k."""
    P1 = P[0]
    P2 = P[1]
    if n == 2:
        return (P1 * P1 - P2) / 2
    P3 = P[2]
    if n == 3:
        return (P1 ** 3 + 2 * P3 - 3 * P1 * P2) / 6
    P4 = P[3]
    if n == 4:
        return (P1 ** 4 - 6 * P4 + 3 * P2 ** 2 - 6 * P2 * P1 ** 2 + 8 * P3 * P1) / 24
    P5 = P[4]
    if n == 5:
        return (P1 ** 5 - 10 * P2 * P1 ** 3 + 15 * P2 ** 2 * P1 + 20 * P3 * P1 ** 2
                - 20 * P3 * P2 - 30 * P1 * P4 + 24 * P5) / 120
    raise ValueError("explicit expansions exist for n = 2..5 only (PAPER.md:140)")


def _partitions(n: int):
    """All (k_1..k_n) >= 0 with sum_i i*k_i = n (the index set of PAPER.md:136)."""
    def rec(i, rem):
        if i > n:
            if rem == 0:
                yield ()
            return
        for k in range(rem // i + 1):
            for rest in rec(i + 1, rem - i * k):
                yield (k,) + rest
    yield from rec(1, n)


def newton_girard_general(P, n: int):
    """General partition formula (Eq. PAPER.md:136, reading Q14 of the garbled LaTeX):

    E_n = sum_{k_1+2k_2+..+nk_n = n} (-1)^(n - sum k_i) prod_{i=1}^{n} P_i^{k_i} / (k_i! i^{k_i})
    """
    total = 0
    for ks in _partitions(n):
        coef = Fraction((-1) ** (n - sum(ks)))
        term = 1
        for i, k in enumerate(ks, start=1):
            coef /= math.factorial(k) * i ** k
            if k:
                term = term * P[i - 1] ** k
        if isinstance(term, Fraction) or isinstance(term, int):
            total = total + coef * term
        else:
            total = total + float(coef) * term
    return total


# --------------------------------------------------------------------------------------
# A4  Coherence factor   (Eq. CF)
# --------------------------------------------------------------------------------------
def coherence_factor(A, B, n_mics: int, eps: float = 1e-30):
    """CF = (sum x)^2 / (N * sum x^2 + eps)  ("a small, positive
    number is typically added to the denominator"; eps reading Q7;
    N = all microphones, reading Q9; CF on x, reading Q8)."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    return (A * A) / (n_mics * B + eps)


def beamform_frame(m, d, p: int, eps: float = 1e-30, chunk: int = 32, alpha=None):
    """All raw images of one frame: DAS (Eq. (2)), DMAS_p (Eqs. (5)/(6)
    PAPER.md:106/116 via ``esp_vieta``), CF, CF-DMAS
    (PAPER.md:177), CF-DAS ("can also be applied to DAS").

    ``m``: [n_mics][T] (fp32 input promoted to float64), ``d``: [n_dirs][n_mics]; with
    ``alpha`` (NEXT-2) the pre-steering interpolates linearly between d and d + 1.
    Returns dict kind -> float64 [n_dirs][T].
    """
    m = np.asarray(m, dtype=np.float64)
    d = np.asarray(d)
    n_dirs = d.shape[0]
    n_mics, T = m.shape
    out = {k: np.empty((n_dirs, T), dtype=np.float64) for k in KIND_NAMES}
    for a0 in range(0, n_dirs, chunk):
        a1 = min(n_dirs, a0 + chunk)
        x = gather(m, d[a0:a1]) if alpha is None else gather_linear(m, d[a0:a1], alpha[a0:a1])
        A = np.sum(x, axis=1)                         # Eq. (2)
        B = np.sum(x * x, axis=1)                     # CF denominator
        s = signed_root(x, p)
        E = esp_vieta([s[:, i, :] for i in range(n_mics)], p)   # Eq. (6)
        cf = coherence_factor(A, B, n_mics, eps)
        out["das"][a0:a1] = A
        out["dmas"][a0:a1] = E
        out["cf"][a0:a1] = cf
        out["cfdmas"][a0:a1] = E * cf
        out["cfdas"][a0:a1] = A * cf
    return out


# --------------------------------------------------------------------------------------
# A5  (band-pass +) envelope   ("absolute value ... then low-pass
#      filtered"; "low-pass filter at 5kHz")
# --------------------------------------------------------------------------------------
def lpf_taps(n_taps: int = 127, cutoff_hz: float = 5000.0, fs: float = 450000.0):
    """Blackman-windowed sinc low-pass (reading Q11), unit DC gain.

    h[n] = (2 fc/fs) sinc((2 fc/fs)(n - (L-1)/2)) w[n],  w[n] = 0.42 - 0.5 cos(2 pi n/(L-1))
    + 0.08 cos(4 pi n/(L-1)),  then h /= sum(h).
    """
    if n_taps < 1 or n_taps % 2 == 0:
        raise ValueError("odd tap count required")
    if not (0.0 < cutoff_hz < fs / 2):
        raise ValueError("0 < cutoff < fs/2 required")
    n = np.arange(n_taps, dtype=np.float64)
    fcn = 2.0 * cutoff_hz / fs
    if n_taps > 1:
        w = 0.42 - 0.5 * np.cos(2 * np.pi * n / (n_taps - 1)) + 0.08 * np.cos(4 * np.pi * n / (n_taps - 1))
    else:
        w = np.ones(1)
    h = fcn * np.sinc(fcn * (n - (n_taps - 1) / 2)) * w
    return h / np.sum(h)


def _fir_same(y, h):
    """Centred FIR (convolution): out[t] = sum_k h[k] y[t + c - k], c = (L-1)/2,
    zeros outside [0, T)."""
    y = np.asarray(y, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    L = h.shape[0]
    c = (L - 1) // 2
    T = y.shape[-1]
    out = np.zeros_like(y)
    for k in range(L):
        sft = c - k                       # out[t] += h[k] * y[t + sft]
        lo, hi = max(0, -sft), min(T, T - sft)
        if lo < hi:
            out[..., lo:hi] += h[k] * y[..., lo + sft:hi + sft]
    return out


def envelope(rows, taps, bp_taps=None, decim: int = 1):
    """Envelope detection along t of each image row: optional
    band-pass FIR (reading Q10, default off) -> |.| -> low-pass FIR -> clamp >= 0
    (reading Q11) -> keep every R-th sample (reading Q12)."""
    y = np.asarray(rows, dtype=np.float64)
    if bp_taps is not None and len(bp_taps) > 0:
        y = _fir_same(y, bp_taps)
    a = np.abs(y)
    e = _fir_same(a, taps)
    e = np.maximum(e, 0.0)
    return e[..., ::decim]
