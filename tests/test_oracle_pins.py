"""Pins of the float64 oracle against things other than itself (CPU only).

Each test names the passage it pins.  The pins are chosen so that a plausible
slip in the oracle (dropped term, wrong sign, wrong index, transposed operand,
wrong rounding) fails at least one of them:

* exact rational identities (brute force over subsets, Eq. (5)) for
  the Vieta E_p, the paper's explicit Newton-Girard forms and the general formula;
* library special cases (numpy.poly for E_k, numpy.convolve for the FIR,
  scipy.signal.firwin for the taps);
* closed forms (coherent plane wave with the table's own delays; DMAS_2 closed
  form of north_star; Eq. (3) literal double sum);
* hand-worked values (tests/golden/worked_examples.json, each with its citation);
* physics independent of the table (echo onsets from workloads.gen line up after
  the oracle's pre-steering), translation invariance, tie rounding.
"""

import itertools
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import dmas_oracle as O
from workloads import gen


# ----------------------------------------------------------------- hand examples
def test_worked_examples(golden):
    for ex in golden["das"]:
        assert sum(ex["x"]) == ex["out"]
        m = np.array(ex["x"], dtype=np.float32)[:, None]
        img = O.beamform_frame(m, np.zeros((1, len(ex["x"])), np.int32), 2)
        assert img["das"][0, 0] == ex["out"]
    for ex in golden["signed_root"]:
        assert O.signed_root(ex["x"], ex["p"]) == pytest.approx(ex["out"], abs=1e-15)
    for ex in golden["power_sums"]:
        s = O.signed_root(ex["x"], ex["p"])
        P = O.power_sums(s, ex["p"])
        assert [float(v) for v in P] == pytest.approx(ex["P"], rel=1e-15)
    for ex in golden["dmas"]:
        s = O.signed_root(ex["x"], ex["p"])
        assert O.esp_vieta(list(s), ex["p"]) == pytest.approx(ex["out"], rel=1e-14)
        m = np.array(ex["x"], dtype=np.float32)[:, None]
        img = O.beamform_frame(m, np.zeros((1, len(ex["x"])), np.int32), ex["p"])
        assert img["dmas"][0, 0] == pytest.approx(ex["out"], rel=1e-14)
    for ex in golden["cf"]:
        x = np.array(ex["x"], dtype=np.float64)
        cf = O.coherence_factor(x.sum(), (x * x).sum(), len(x), eps=0.0)
        assert float(cf) == pytest.approx(ex["out"], abs=1e-15)


def test_chirp_and_eta_examples(golden):
    g = golden["chirp_samples"]
    assert gen.chirp_samples(g["fs"]).shape[0] == g["n"]
    for ex in golden["eta"]:
        assert 10.0 ** (-ex["snr_db"] / 20.0) == pytest.approx(ex["eta"], rel=1e-12)


# ----------------------------------------------------------------- A1 delay table
def test_delay_worked_example(golden):
    ex = golden["delay"][0]
    d, v = O.delay_table([ex["mic"]], [[ex["az"], ex["el"]]], ex["fs"], ex["c"], return_exact=True)
    assert abs(v[0, 0]) == pytest.approx(ex["abs_v_samples"], abs=5e-4)
    assert abs(v[0, 0]) / ex["fs"] == pytest.approx(ex["abs_tau_s"], rel=1e-4)
    assert d[0, 0] == ex["d"]


def test_delay_broadside_planar_is_zero():
    """planar array in the y-z plane, direction +x -> all delays 0."""
    mic = gen.disk_array(32, seed=7)
    d = O.delay_table(mic, [[0.0, 0.0]], 450e3, 343.0)
    assert np.all(d == 0)


def test_delay_ties_to_even():
    """Reading Q4: nearest sample, ties to even (fs/c = 1 makes v exact)."""
    mics = [[-0.5, 0, 0], [-1.5, 0, 0], [-2.5, 0, 0], [0.5, 0, 0], [-2.4, 0, 0], [-2.6, 0, 0]]
    d = O.delay_table(mics, [[0.0, 0.0]], 343.0, 343.0)
    assert list(d[0]) == [0, 2, 2, 0, 2, 3]


def test_delay_translation_invariance():
    """shifting mics and reference by one vector leaves delays unchanged."""
    mic = gen.disk_array(16, seed=3)
    dirs = gen.az_el_grid(9, 80.0, 7, 50.0)
    shift = np.array([0.25, -0.5, 0.125])          # exact binary fractions: no new rounding in p - r
    d0 = O.delay_table(mic, dirs, 450e3, 343.0)
    d1 = O.delay_table(mic + shift, dirs, 450e3, 343.0, reference=shift)
    # p - r is exact only when the shift is representable alongside p; allow a
    # rounding flip only where v sits within 1e-9 of a half-integer (none expected)
    assert np.array_equal(d0, d1)


def test_delay_bound_and_axes():
    """|d| <= ceil(aperture fs/c); az moves along +y, el along +z (reading Q3)."""
    mic = gen.ula(8)                                  # on the y axis
    d = O.delay_table(mic, gen.az_grid_deg([-90, 0, 90]), 450e3, 343.0)
    ap = np.max(np.abs(mic[:, 1]))
    assert np.all(np.abs(d) <= math.ceil(ap * 450e3 / 343.0))
    assert np.all(d[1] == 0)                          # broadside
    assert np.array_equal(d[0], -d[2])                # mirror
    # az = +90 deg: u = +y, the +y-most mic hears first -> most negative delay
    assert d[2, -1] == d[2].min() < 0
    dz = O.delay_table([[0, 0, 0.05]], [[0.0, math.radians(90.0)]], 450e3, 343.0)
    assert dz[0, 0] == round(-0.05 * 450e3 / 343.0)


def test_delay_aligns_independent_echo_physics():
    """Pre-steering with the oracle table lines up echoes synthesised analytically by
    workloads.gen (independent of the table): per-mic envelope peak of the
    matched-filtered signal, after gather, at the same sample within +-1."""
    mic = gen.disk_array(32, seed=7)
    az, el = math.radians(23.0), math.radians(-11.0)
    R = 0.5                                          # onset sample 1312 < T
    m = gen.frame(mic, [(az, el, R, 1.0)], 2048)
    d = O.delay_table(mic, [[az, el]], gen.FS, gen.C_SOUND)
    x = O.gather(m, d)[0]
    peaks = np.argmax(np.abs(x), axis=1)
    expect = round(2 * R / gen.C_SOUND * gen.FS)
    assert np.all(np.abs(peaks - expect) <= 1), (peaks, expect)
    # and a sign flip would scatter them
    xb = O.gather(m, -d)[0]
    assert np.ptp(np.argmax(np.abs(xb), axis=1)) > 10


# ----------------------------------------------------------------- A2 gather
def test_gather_hand_example():
    m = np.arange(1, 9, dtype=np.float32).reshape(2, 4)     # [[1,2,3,4],[5,6,7,8]]
    d = np.array([[1, -2], [0, 5]], dtype=np.int32)
    x = O.gather(m, d)
    assert x[0].tolist() == [[2, 3, 4, 0], [0, 0, 5, 6]]
    assert x[1].tolist() == [[1, 2, 3, 4], [0, 0, 0, 0]]


# ----------------------------------------------------------------- E_p: Vieta vs brute force (exact)
def _rand_fracs(rng, n):
    return [Fraction(rng.randint(-50, 50), rng.randint(1, 20)) for _ in range(n)]


def test_vieta_equals_bruteforce_exact():
    """Eq. (6) PAPER.md:116 == Eq. (5), exactly in rationals."""
    rng = random.Random(1)
    for p in range(1, 7):
        for N in range(p, 10):
            for _ in range(10):
                s = _rand_fracs(rng, N)
                assert O.esp_vieta(s, p) == O.brute_force_esp(s, p)


def test_newton_girard_explicit_exact():
    """Explicit forms n = 2..5 and the general partition formula
     equal brute-force E_n exactly (rationals)."""
    rng = random.Random(2)
    for n in range(2, 8):
        for N in range(n, 10):
            for _ in range(6):
                s = _rand_fracs(rng, N)
                P = [sum(v ** k for v in s) for k in range(1, n + 1)]
                e = O.brute_force_esp(s, n)
                assert O.newton_girard_general(P, n) == e
                if n <= 5:
                    assert O.newton_girard_explicit(P, n) == e


def test_vieta_matches_numpy_poly():
    """Library special case: numpy.poly(s) = coefficients of prod(z - s_i) = sum (-1)^k E_k z^(N-k)."""
    rng = np.random.default_rng(3)
    for N in (5, 12, 32):
        s = rng.uniform(-1, 1, N)
        c = np.poly(s)
        for p in range(1, 6):
            assert O.esp_vieta(list(s), p) == pytest.approx((-1) ** p * c[p], rel=1e-10, abs=1e-12)


def test_dmas2_eq3_and_closed_form():
    """Eq. (3) PAPER.md:97 literal double sum == Vieta E_2 of signed roots == the
    closed form ((sum sgn sqrt|x|)^2 - sum |x|)/2 (north_star), N = 32."""
    rng = np.random.default_rng(4)
    for _ in range(300):
        x = rng.uniform(-1, 1, 32)
        eq3 = O.dmas_pairwise_eq3(x)
        s = O.signed_root(x, 2)
        vieta = O.esp_vieta(list(s), 2)
        closed = (np.sum(np.sign(x) * np.sqrt(np.abs(x))) ** 2 - np.sum(np.abs(x))) / 2
        assert vieta == pytest.approx(eq3, rel=1e-9, abs=1e-12)
        assert closed == pytest.approx(eq3, rel=1e-9, abs=1e-12)


def test_float_vieta_vs_bruteforce():
    """p in 2..6, N in p..10, random slices in [-1,1], 1e-9 relative."""
    rng = np.random.default_rng(5)
    for p in range(2, 7):
        for N in range(p, 11):
            for _ in range(8):
                x = rng.uniform(-1, 1, N)
                s = list(O.signed_root(x, p))
                assert O.esp_vieta(s, p) == pytest.approx(O.brute_force_esp(s, p), rel=1e-9, abs=1e-12)


# ----------------------------------------------------------------- CF
def test_cf_properties():
    """CF in [0,1] (Cauchy-Schwarz), scale invariance, constant -> 1."""
    rng = np.random.default_rng(6)
    X = rng.uniform(-1, 1, (2000, 16))
    A, B = X.sum(1), (X * X).sum(1)
    cf = O.coherence_factor(A, B, 16, eps=0.0)
    assert np.all(cf >= 0) and np.all(cf <= 1 + 1e-15)
    for lam in (1e-3, 1.0, 1e3):
        cfl = O.coherence_factor(lam * A, lam * lam * B, 16, eps=0.0)
        np.testing.assert_allclose(cfl, cf, rtol=1e-9)
    assert float(O.coherence_factor(0.0, 0.0, 8)) == 0.0          # all-zero slice, eps > 0


def test_power_sums_signed_and_newton_girard_route():
    """P_k = sum_i s_i^k keeps the signs of odd powers (Eq. PAPER.md:131): s = (-1, 2) gives
    (P1, P2, P3) = (1, 5, 7) by hand; and the paper's Newton-Girard expansion of those sums
     reproduces E_3 of a mixed-sign set, e.g. E_3(-1, 2, 3) = -6 (hand value)."""
    assert [float(v) for v in O.power_sums(np.array([-1.0, 2.0]), 3)] == [1.0, 5.0, 7.0]
    s = np.array([-1.0, 2.0, 3.0])
    assert float(O.newton_girard_explicit(O.power_sums(s, 3), 3)) == pytest.approx(-6.0, abs=1e-12)
    assert float(O.esp_vieta(list(s), 3)) == -6.0


def test_cf_default_eps_is_negligible():
    """CF's guard is "a small, positive number" (reading Q7: 1e-30): a perfectly
    coherent slice of tiny amplitude (x_i = 1e-9, N B = 6.4e-17) still has CF = 1 to ~1e-14, and
    through beamform_frame's default the same holds on a one-pixel frame."""
    x = np.full(8, 1e-9)
    assert float(O.coherence_factor(x.sum(), (x * x).sum(), 8)) == pytest.approx(1.0, abs=1e-12)
    img = O.beamform_frame(np.full((8, 1), 1e-9, np.float32), np.zeros((1, 8), np.int32), 2)
    assert float(img["cf"][0, 0]) == pytest.approx(1.0, abs=1e-12)


# ----------------------------------------------------------------- beamform_frame against per-pixel brute force
def test_beamform_frame_bruteforce_pixels():
    """Whole chain (gather -> roots -> E_p, A, B, CF) against an independent per-pixel
    evaluation written here from Eqs. (1), (2), (5), CF."""
    rng = np.random.default_rng(7)
    n_mics, T, n_dirs = 6, 24, 4
    m = rng.standard_normal((n_mics, T)).astype(np.float32)
    d = rng.integers(-5, 6, size=(n_dirs, n_mics)).astype(np.int32)
    for p in (2, 3, 4, 5):
        img = O.beamform_frame(m, d, p)
        for a in range(n_dirs):
            for t in range(T):
                x = [float(m[i, t + d[a, i]]) if 0 <= t + d[a, i] < T else 0.0 for i in range(n_mics)]
                s = [math.copysign(abs(v) ** (1.0 / p), v) if v != 0 else 0.0 for v in x]
                E = sum(math.prod(c) for c in itertools.combinations(s, p))
                A = sum(x)
                B = sum(v * v for v in x)
                cf = A * A / (n_mics * B + 1e-30)
                assert img["dmas"][a, t] == pytest.approx(E, rel=1e-9, abs=1e-12)
                assert img["das"][a, t] == pytest.approx(A, rel=1e-12, abs=1e-12)
                assert img["cf"][a, t] == pytest.approx(cf, rel=1e-12, abs=1e-15)
                assert img["cfdmas"][a, t] == pytest.approx(E * cf, rel=1e-9, abs=1e-12)
                assert img["cfdas"][a, t] == pytest.approx(A * cf, rel=1e-12, abs=1e-12)


def test_coherent_plane_wave_closed_forms():
    """m_i[t] = w[t - d_i] built from the table's own delays: at interior samples
    CF = 1, DAS = N w, DMAS_p = C(N,p) w (odd p) or C(N,p)|w| (even p)."""
    mic = gen.disk_array(16, seed=9)
    dirs = gen.az_el_grid(5, 60.0, 3, 30.0)
    d = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND)
    T = 256
    rng = np.random.default_rng(8)
    w = rng.uniform(-1, 1, T + 400)
    a = 7                                            # steer at direction 7
    m = np.zeros((16, T), dtype=np.float64)
    for i in range(16):
        for t in range(T):
            m[i, t] = w[200 + t - d[a, i]]
    m32 = m.astype(np.float32)
    wt = np.array([np.float32(w[200 + t]) for t in range(T)], dtype=np.float64)
    lo, hi = 80, T - 80
    for p in (2, 3, 4, 5):
        img = O.beamform_frame(m32, d[a:a + 1], p)
        np.testing.assert_allclose(img["cf"][0, lo:hi], 1.0, rtol=1e-12)
        np.testing.assert_allclose(img["das"][0, lo:hi], 16 * wt[lo:hi], rtol=1e-12)
        ref = math.comb(16, p) * (wt[lo:hi] if p % 2 else np.abs(wt[lo:hi]))
        np.testing.assert_allclose(img["dmas"][0, lo:hi], ref, rtol=1e-9, atol=1e-12)


def test_scaling_sign_permutation():
    """S(lam x) = lam S(x) (lam > 0), S(-x) = (-1)^p S(x), mic permutation invariance."""
    rng = np.random.default_rng(10)
    m = rng.standard_normal((7, 40))
    d = rng.integers(-4, 5, size=(3, 7)).astype(np.int32)
    perm = rng.permutation(7)
    for p in (2, 3, 4, 5):
        base = O.beamform_frame(m, d, p)
        sc = O.beamform_frame(2.5 * m, d, p)
        ng = O.beamform_frame(-m, d, p)
        pm = O.beamform_frame(m[perm], d[:, perm], p)
        np.testing.assert_allclose(sc["dmas"], 2.5 * base["dmas"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(ng["dmas"], (-1) ** p * base["dmas"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(pm["dmas"], base["dmas"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(pm["cf"], base["cf"], rtol=1e-9, atol=1e-12)


def test_zero_input_zero_output():
    img = O.beamform_frame(np.zeros((4, 10)), np.zeros((2, 4), np.int32), 3)
    for k in oracle.KIND_NAMES:
        assert np.all(img[k] == 0)


# ----------------------------------------------------------------- A5 envelope
def test_lpf_taps_match_scipy_firwin():
    """Blackman windowed sinc, unit DC gain (reading Q11) == scipy.signal.firwin."""
    import scipy.signal as ss
    h = O.lpf_taps(127, 5000.0, 450e3)
    ref = ss.firwin(127, 5000.0, window="blackman", fs=450e3)
    np.testing.assert_allclose(h, ref, rtol=0, atol=1e-15)
    assert h.sum() == pytest.approx(1.0, abs=1e-14)
    np.testing.assert_allclose(h, h[::-1], rtol=0, atol=1e-16)   # linear phase (symmetric)


def test_fir_matches_numpy_convolve():
    rng = np.random.default_rng(11)
    y = rng.standard_normal((3, 300))
    for L in (1, 5, 127):
        h = rng.standard_normal(L)
        out = O._fir_same(y, h)
        for r in range(3):
            np.testing.assert_allclose(out[r], np.convolve(y[r], h, mode="same"), rtol=1e-12, atol=1e-12)


def test_envelope_properties(golden):
    g = golden["envelope_tone"]
    h = O.lpf_taps(127, g["cutoff_hz"], g["fs"])
    T = 4000
    t = np.arange(T)
    tone = np.sin(2 * np.pi * g["f_hz"] * t / g["fs"])
    e = O.envelope(tone[None], h)[0]
    assert e[200:-200].mean() == pytest.approx(g["mean"], rel=g["rel_tol"])
    # DC gain 1 in the interior (>= 63 samples from either edge), zero -> zero, >= 0
    c = O.envelope(np.full((1, 500), -0.75), h)[0]
    np.testing.assert_allclose(c[63:-63], 0.75, rtol=1e-13)
    assert c[0] < 0.75
    assert np.all(O.envelope(np.zeros((2, 50)), h) == 0)
    rng = np.random.default_rng(12)
    r = O.envelope(rng.standard_normal((4, 300)), h)
    assert np.all(r >= 0)
    # decimation keeps every R-th sample, ceil(T/R) of them
    full = O.envelope(rng.standard_normal((2, 301)), h)
    assert O.envelope(np.zeros((1, 301)), h, decim=4).shape == (1, 76)
    # identity band-pass [1] changes nothing
    y = rng.standard_normal((2, 200))
    np.testing.assert_array_equal(O.envelope(y, h, bp_taps=[1.0]), O.envelope(y, h))
    assert full.shape == (2, 301)


def test_envelope_impulse_response_clamp():
    """Clamp >= 0 (reading Q11, "clamped to be non-negative"), pinned by a closed
    form: a unit impulse at t0 through the centred FIR gives h[k] at t = t0 + k - c (convolution of
    a delta with h is h, numpy.convolve), so the envelope is max(h[k], 0) there and 0 elsewhere.
    The 127-tap Blackman low-pass has 34 negative taps: a rectifier |.| instead of the clamp would
    return |h[k]| at those samples, a missing clamp h[k] < 0."""
    h = O.lpf_taps(127, 5000.0, 450e3)
    neg = np.flatnonzero(h < 0)
    assert len(neg) == 34
    T, t0, c = 400, 150, 63
    y = np.zeros((1, T))
    y[0, t0] = 1.0
    e = O.envelope(y, h)[0]
    expect = np.zeros(T)
    expect[t0 - c:t0 - c + 127] = np.maximum(np.convolve([1.0], h), 0.0)
    np.testing.assert_array_equal(e, expect)
    assert np.all(e[t0 - c + neg] == 0.0)
    # a negative impulse gives the same envelope (|.| comes before the low-pass)
    np.testing.assert_array_equal(O.envelope(-y, h)[0], e)


def test_envelope_bandpass_orientation():
    """The band-pass is a centred convolution (out[t] = sum_k h[k] y[t + c - k]),
    pinned with an asymmetric 3-tap filter [0, 0, 1] (c = 1): out[t] = y[t - 1], a one-sample
    delay -- numpy.convolve(mode="same") agrees; a correlation would advance by one sample instead.
    The identity low-pass [1] leaves |y| visible."""
    rng = np.random.default_rng(13)
    y = rng.standard_normal((2, 50))
    bp = np.array([0.0, 0.0, 1.0])
    out = O.envelope(y, np.array([1.0]), bp_taps=bp)
    expect = np.zeros_like(y)
    expect[:, 1:] = np.abs(y[:, :-1])
    np.testing.assert_array_equal(out, expect)
    for r in range(2):
        np.testing.assert_array_equal(out[r], np.abs(np.convolve(y[r], bp, mode="same")))
    # and a random asymmetric band-pass before the 127-tap low-pass matches numpy.convolve twice
    bp2 = rng.standard_normal(31)
    h = O.lpf_taps(127, 5000.0, 450e3)
    y = rng.standard_normal((2, 300))
    ref = np.stack([np.maximum(np.convolve(np.abs(np.convolve(y[r], bp2, mode="same")), h, mode="same"), 0)
                    for r in range(2)])
    np.testing.assert_allclose(O.envelope(y, h, bp_taps=bp2), ref, rtol=1e-12, atol=1e-14)


# ----------------------------------------------------------------- pipeline trend
def test_pipeline_peak_and_dynamic_range_trend():
    """Noise-free 32-mic PSF scan (az -90..90 step 2, reflector at az 10 deg, sample
    1312): every kind peaks at the reflector; the directional dynamic range (peak vs
    max response > 20 deg off the peak) rises DAS -> DMAS2 -> ... -> DMAS5 and CF raises
    it for every order ("higher dynamic range for increasing orders"
    ... "CF post-processing step further increases")."""
    mic = gen.disk_array(32, seed=7)
    dirs = gen.az_grid_deg(np.arange(-90, 91, 2))
    m = gen.frame(mic, [(math.radians(10.0), 0.0, 0.5, 1.0)], 1536)
    d = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND)
    h = O.lpf_taps()
    az = np.rad2deg(dirs[:, 0])

    def dyn_range(img):
        env = O.envelope(img, h)
        a, t = np.unravel_index(np.argmax(env), env.shape)
        assert round(az[a]) == 10 and abs(t - 1312) <= 2
        prof = env.max(axis=1)
        return 20 * np.log10(prof[a] / np.max(prof[np.abs(az - az[a]) > 20]))

    prev = dyn_range(O.beamform_frame(m, d, 2)["das"])
    for p in (2, 3, 4, 5):
        img = O.beamform_frame(m, d, p)
        dr = dyn_range(img["dmas"])
        assert dr > prev
        assert dyn_range(img["cfdmas"]) > dr
        prev = dr


# ----------------------------------------------------------------- A0 matched filter (NEXT-1)
def test_matched_filter_worked_examples():
    """the emitted signal itself peaks at 1 at lag 0; a copy delayed by 100
    samples peaks at sample 100 (>= 0.999); zeros stay zeros."""
    w = gen.chirp_samples()
    L = len(w)
    y = O.matched_filter(np.concatenate([w, np.zeros(L)]), w, 1)
    assert y[0] == pytest.approx(1.0, rel=1e-12)
    raw = np.zeros(400 + 2 * L)
    raw[100:100 + L] = w
    y = O.matched_filter(raw, w, 400)
    assert int(np.argmax(y)) == 100 and y[100] >= 0.999
    assert np.all(O.matched_filter(np.zeros((2, 50 + L)), w, 51) == 0)


def test_matched_filter_definition_and_library_cases():
    """Brute force on a tiny case, numpy.correlate ('valid'), linearity, and the generator's
    independent FFT implementation."""
    rng = np.random.default_rng(70)
    w = rng.standard_normal(7)
    raw = rng.standard_normal((3, 40))
    T = 40 - 7 + 1
    y = O.matched_filter(raw, w, T)
    E = float(np.sum(w * w))
    for c in range(3):
        brute = [sum(w[k] * raw[c, t + k] for k in range(7)) / E for t in range(T)]
        np.testing.assert_allclose(y[c], brute, rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(y[c], np.correlate(raw[c], w, "valid") / E, rtol=1e-12, atol=1e-13)
    raw2 = rng.standard_normal((3, 40))
    np.testing.assert_allclose(O.matched_filter(2 * raw - 3 * raw2, w, T), 2 * y - 3 * O.matched_filter(raw2, w, T),
                               rtol=1e-12, atol=1e-12)
    mic = gen.disk_array(8, 0.05, 5e-3, seed=2)
    r = gen.raw_frame(mic, [(0.3, 0.1, 0.6, 1.0)], 800, snr_db=0.0, seed=1)
    np.testing.assert_allclose(O.matched_filter(r, gen.chirp_samples(), 800), gen.matched_filter(r, 800),
                               rtol=1e-9, atol=1e-9)


# ----------------------------------------------------------------- NEXT-2 fractional-delay pre-steering
def test_linear_delay_table_and_gather():
    """d0 = floor(v), alpha = v - d0 in [0,1), d0 + alpha = the exact delay; alpha = 0 reduces to the
    integer gather; linear interpolation reproduces a linear ramp exactly; alpha = 1/2 averages."""
    mic = gen.disk_array(16, seed=3)
    dirs = gen.az_el_grid(7, 70.0, 5, 40.0)
    d0, al = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND, mode="linear")
    _, v = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND, return_exact=True)
    assert np.all((al >= 0) & (al < 1))
    np.testing.assert_allclose(d0 + al, v, rtol=0, atol=1e-12)
    assert np.array_equal(d0, np.floor(v).astype(np.int32))
    rng = np.random.default_rng(90)
    m = rng.standard_normal((16, 300))
    np.testing.assert_array_equal(O.gather_linear(m, d0, np.zeros_like(al)), O.gather(m, d0))
    ramp = np.tile(0.25 * np.arange(300.0) - 3.0, (16, 1))
    x = O.gather_linear(ramp, d0, al)
    t = np.arange(300.0)
    inside = (t[None, None, :] + d0[:, :, None] >= 0) & (t[None, None, :] + d0[:, :, None] + 1 < 300)
    exp = 0.25 * (t[None, None, :] + d0[:, :, None] + al[:, :, None]) - 3.0
    np.testing.assert_allclose(x[inside], exp[inside], rtol=1e-12, atol=1e-12)
    half = O.gather_linear(m, d0, np.full_like(al, 0.5))
    np.testing.assert_allclose(half, 0.5 * (O.gather(m, d0) + O.gather(m, d0 + 1)), rtol=1e-13)


def test_linear_presteer_aligns_physical_plane_wave():
    """A fractional plane wave (analytic echoes at non-integer delays) is aligned better by linear
    interpolation than by nearest-sample steering: higher CF at the echo (SPEC.md:217 rationale)."""
    mic = gen.disk_array(32, seed=7)
    az, el = math.radians(17.0), math.radians(-9.0)
    m = gen.frame(mic, [(az, el, 0.5, 1.0)], 1536)
    d = O.delay_table(mic, [[az, el]], gen.FS, gen.C_SOUND)
    d0, al = O.delay_table(mic, [[az, el]], gen.FS, gen.C_SOUND, mode="linear")
    cf_near = O.beamform_frame(m, d, 2)["cf"][0, 1300:1325].max()
    cf_lin = O.beamform_frame(m, d0, 2, alpha=al)["cf"][0, 1300:1325].max()
    assert cf_lin > cf_near > 0.5


def test_hex_lattice_counts():
    """5 mm hexagonal lattice, radius 1 cm -> 19 microphones (paper's lower
    bound); radius 2.4 mm -> 1.  At 6 cm a site-centred lattice gives 517, not the
    paper's "513" (513 = 3 mod 6 cannot come from a 6-fold-symmetric
    site-centred lattice) — recorded, not matched."""
    assert len(gen.hex_array(0.0024)) == 1
    assert len(gen.hex_array(0.01)) == 19
    assert len(gen.hex_array(0.06)) == 517
    a = gen.hex_array(0.03)
    assert np.allclose(a[:, 0], 0) and np.allclose(a.mean(axis=0), 0, atol=1e-12)
    dist = np.linalg.norm(a[:, None, 1:] - a[None, :, 1:], axis=-1) + np.eye(len(a))
    assert np.isclose(dist.min(), 5e-3)
