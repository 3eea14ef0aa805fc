"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on identical
seeded inputs.  Bar (BASELINE.json north_star): delay tables bit-exact; every image kind,
frame and stage within max|gpu - oracle| <= 1e-4 * max|oracle|."""

import math

import numpy as np
import pytest

from oracle import dmas_oracle as O
from workloads import gen

pytestmark = pytest.mark.gpu

TOL = 1e-4           # relative to the image peak (north_star)
KINDS = ("das", "dmas", "cfdmas", "cfdas", "cf")


@pytest.fixture(scope="module")
def dm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2511_09165_b200 import dmas
    return dmas


def run_gpu(dm, mic, dirs, fs, c, p, signals, what, n_samples=None, **kw):
    import torch
    F = signals.shape[0]
    plan = dm.Plan(mic, dirs, fs, c, p, n_samples or signals.shape[2], max_frames=max(1, F), **kw)
    x = torch.from_numpy(np.ascontiguousarray(signals)).cuda()
    res = plan.beamform(x, what)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in res.items()}
    return plan, out


def oracle_images(mic, dirs, fs, c, p, signals, kinds=KINDS, env_kinds=(), lp_taps=127, cutoff=5000.0,
                  bp=None, decim=1, d=None, eps=1e-30):
    if d is None:
        d = O.delay_table(mic, dirs, fs, c)
    h = O.lpf_taps(lp_taps, cutoff, fs) if env_kinds else None
    out = {}
    for f in range(signals.shape[0]):
        img = O.beamform_frame(signals[f], d, p, eps=eps)
        for k in kinds:
            out.setdefault(("raw", k), []).append(img[k])
        for k in env_kinds:
            out.setdefault(("env", k), []).append(O.envelope(img[k], h, bp_taps=bp, decim=decim))
    return {k: np.stack(v) for k, v in out.items()}


def assert_parity(gpu, ref, label="", zero_scale=None):
    """max|gpu - ref| <= 1e-4 * max|ref| per frame.  When the oracle image is exactly zero the
    relative criterion is undefined; fp32 Newton-Girard then leaves a rounding residue of the
    order of the inputs, so the bound is taken relative to `zero_scale` (an upper bound of
    |image| from the input amplitudes) when given, else 1e-30."""
    assert gpu.shape == ref.shape, (label, gpu.shape, ref.shape)
    for f in range(ref.shape[0]):
        peak = float(np.max(np.abs(ref[f])))
        err = float(np.max(np.abs(gpu[f].astype(np.float64) - ref[f])))
        bound = TOL * peak if peak > 0 else (TOL * zero_scale if zero_scale else 1e-30)
        assert np.all(np.isfinite(gpu[f])), label
        assert err <= bound, f"{label} frame {f}: max err {err:.3e} > {bound:.3e} (peak {peak:.3e})"


def what_all(dm, env=True):
    return dm.RAW(dm.KIND_ALL) | (dm.ENV(dm.KIND_ALL) if env else 0)


# ------------------------------------------------------------------ A1 bit-exact delay tables
@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5", "paper3601"])
def test_delay_table_bitexact(dm, name):
    if name == "paper3601":          # 3601 azimuths, 0.05 deg, el 0, 32-mic eRTIS-like
        mic, dirs = gen.disk_array(32, seed=7), gen.az_grid_deg(np.linspace(-90, 90, 3601))
    elif name == "C4":
        mic, dirs = gen.disk_array(64, 0.10, 4e-3, seed=11), gen.az_el_grid(128, 90.0, 128, 60.0)
    elif name == "C5":
        mic, dirs = gen.disk_array(32, seed=7), gen.az_el_grid(128, 90.0, 128, 60.0)
    elif name == "C2":
        mic, dirs = gen.disk_array(32, seed=7), gen.az_el_grid(60, 90.0, 30, 45.0)
    else:
        mic, dirs = gen.ula(8), gen.az_grid_deg(np.arange(-90, 91, 2))
    plan = dm.Plan(mic, dirs, gen.FS, gen.C_SOUND, 2, 64)
    d_gpu = plan.delay_table()
    d_ref, v = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND, return_exact=True)
    assert np.array_equal(d_gpu, d_ref)
    margin = float(np.min(np.abs(np.abs(v - np.floor(v)) - 0.5)))
    assert margin > 1e-9        # no near-ties: the bit-exact claim is not luck
    assert plan.info["d_min"] == d_ref.min() and plan.info["d_max"] == d_ref.max()


def test_delay_table_reference_point_and_ties(dm):
    mics = np.array([[-0.5, 0, 0], [-1.5, 0, 0], [-2.5, 0, 0], [0.5, 0, 0], [-2.4, 0.1, 0], [-2.6, 0, 0.1]])
    plan = dm.Plan(mics, [[0.0, 0.0]], 343.0, 343.0, 2, 16, lp_taps=0)
    assert plan.delay_table().tolist() == O.delay_table(mics, [[0.0, 0.0]], 343.0, 343.0).tolist()
    mic = gen.disk_array(16, seed=3)
    dirs = gen.az_el_grid(9, 80.0, 7, 50.0)
    ref = np.array([0.01, -0.02, 0.005])
    plan = dm.Plan(mic, dirs, gen.FS, gen.C_SOUND, 2, 16, reference_xyz=ref)
    assert np.array_equal(plan.delay_table(), O.delay_table(mic, dirs, gen.FS, gen.C_SOUND, reference=ref))


# ------------------------------------------------------------------ slice harness (broadside, zero delays)
def _slice_plan(dm, n, p, T):
    mic = np.stack([np.zeros(n), 0.003 * np.arange(n) - 0.0015 * (n - 1), np.zeros(n)], axis=1)
    return dm.Plan(mic, [[0.0, 0.0]], gen.FS, gen.C_SOUND, p, T)


def test_slice_harness_worked_examples(dm, golden):
    """Array in the y-z plane + one broadside direction => every delay is 0 and x_i(t) = m_i[t]:
    each sample column is an independent slice.  SPEC worked examples on the GPU."""
    import torch
    cases = [(np.array([1, 4, 9.0]), 2, {"dmas": 11.0, "das": 14.0}),
             (np.array([1, 8, 27, 64.0]), 3, {"dmas": 50.0, "das": 100.0}),
             (np.array([1, 0, 0, 0.0]), 2, {"cf": 0.25}),
             (np.array([1, -1.0]), 2, {"cf": 0.0, "dmas": -1.0})]
    for x, p, exp in cases:
        plan = _slice_plan(dm, len(x), p, 1)
        assert np.all(plan.delay_table() == 0)
        sig = torch.tensor(x, dtype=torch.float32).reshape(1, len(x), 1).cuda()
        res = plan.beamform(sig, dm.RAW(dm.KIND_ALL))
        for k, v in exp.items():
            assert float(res[("raw", k)].item()) == pytest.approx(v, rel=1e-6, abs=1e-6), (x, p, k)


def test_slice_harness_random_bruteforce(dm):
    """Random slices (N <= 10, p <= 5) against Eq. (5) brute force, plus S(lam x) = lam S(x)
    and S(-x) = (-1)^p S(x) on the GPU."""
    import torch
    rng = np.random.default_rng(21)
    for p in (2, 3, 4, 5):
        for n in (p, 7, 10):
            T = 300
            x = rng.uniform(-1, 1, (n, T)).astype(np.float32)
            plan = _slice_plan(dm, n, p, T)
            sig = torch.from_numpy(x[None]).cuda()
            g = plan.beamform(sig, dm.RAW(dm.KIND_DMAS))[("raw", "dmas")].cpu().numpy()[0, 0]
            g2 = plan.beamform(2.0 * sig, dm.RAW(dm.KIND_DMAS))[("raw", "dmas")].cpu().numpy()[0, 0]
            gn = plan.beamform(-sig, dm.RAW(dm.KIND_DMAS))[("raw", "dmas")].cpu().numpy()[0, 0]
            ref = np.array([O.brute_force_esp(list(O.signed_root(x[:, t].astype(np.float64), p)), p)
                            for t in range(T)])
            peak = np.max(np.abs(ref))
            assert np.max(np.abs(g - ref)) <= 1e-5 * peak
            assert np.max(np.abs(g2 - 2 * ref)) <= 1e-5 * 2 * peak
            assert np.max(np.abs(gn - (-1) ** p * ref)) <= 1e-5 * peak


# ------------------------------------------------------------------ random multi-tile / ragged cases
@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_random_multi_tile_all_kinds(dm, p):
    """Several psi tiles (70 dirs = 2 full + ragged), several t tiles (700 = 2 full + ragged),
    3 frames, 11 mics, every kind, raw + envelope."""
    mic = gen.disk_array(11, 0.08, 5e-3, seed=30 + p)
    dirs = gen.az_el_grid(10, 80.0, 7, 50.0)
    sig = gen.random_signals(3, 11, 700, seed=40 + p, sparsity=0.1)
    plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, p, sig, what_all(dm))
    ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, p, sig, env_kinds=KINDS)
    for key in ref:
        assert_parity(g[key], ref[key], f"p={p} {key}")


# ------------------------------------------------------------------ BASELINE.json configs
def _config_parity(dm, name, p=None, env=True):
    cfg = gen.config(name)
    p = p or cfg["order"]
    plan, g = run_gpu(dm, cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], p, cfg["signals"], what_all(dm, env))
    ref = oracle_images(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], p, cfg["signals"],
                        env_kinds=KINDS if env else ())
    for key in ref:
        assert_parity(g[key], ref[key], f"{name} p={p} {key}")


def test_config_C1(dm):
    _config_parity(dm, "C1")


def test_config_C2(dm):
    _config_parity(dm, "C2")


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_config_C3_order_sweep(dm, p):
    _config_parity(dm, "C3", p=p)


def _assert_whole_frames(res, label):
    """res from tests/_oracle_pool.compare_frames: the north_star bar over every pixel of each frame."""
    assert res
    for (stage, kind, f), (err, peak, finite) in sorted(res.items()):
        assert finite, (label, stage, kind, f)
        assert peak > 0, (label, stage, kind, f)
        assert err <= TOL * peak, f"{label} {stage}/{kind} frame {f}: max err {err:.3e} > {TOL * peak:.3e}"


def test_config_C4_whole_frame_all_kinds(dm):
    """C4 (64 mics, 16,384 directions, T = 8192, p = 3) frame 0, EVERY kind raw and envelope, over the
    whole frame (134 M pixels per image) against the oracle (process pool over direction chunks)."""
    import torch
    from _oracle_pool import compare_frames
    cfg = gen.config("C4", frames=1)
    sig = cfg["signals"]
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 3, cfg["T"], max_frames=1)
    res = plan.beamform(torch.from_numpy(sig).cuda(), what_all(dm))
    torch.cuda.synchronize()
    gpu = {k: v.cpu().numpy() for k, v in res.items()}
    del res
    d = plan.delay_table()
    assert np.array_equal(d, O.delay_table(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"]))
    _assert_whole_frames(compare_frames(sig, d, 3, gpu, [0], chunk=128), "C4")


def test_config_C5_frame_all_kinds_whole_frame(dm):
    """C5 frame 200 (3 reflectors advanced 0.2 m, its own noise), every kind raw and envelope, over
    the whole 67 M-pixel frame against the oracle."""
    import torch
    from _oracle_pool import compare_frames
    cfg = gen.config("C5", frames=201)
    sig = np.ascontiguousarray(cfg["signals"][200:201])
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=1)
    res = plan.beamform(torch.from_numpy(sig).cuda(), what_all(dm))
    torch.cuda.synchronize()
    gpu = {k: v.cpu().numpy() for k, v in res.items()}
    del res
    d = plan.delay_table()
    r = compare_frames(sig, d, 2, gpu, [0])
    assert len(r) == 10
    _assert_whole_frames(r, "C5 f200")


def test_config_C5_bench_launch_whole_frames(dm):
    """C5 in the launch configuration bench.py times: one call over 256 frames, CF-DMAS2 envelope
    only (the raw image goes through the plan scratch in internal frame chunks).  Frames
    {0, 128, 255} are compared over the WHOLE frame (67 M pixels) with the oracle; then the same three
    frames are beamformed with the raw CF-DMAS image requested too: raw parity over the whole frame,
    and the envelope of that request is bitwise the bench launch's."""
    import torch
    from _oracle_pool import compare_frames
    cfg = gen.config("C5")
    sig = cfg["signals"]
    frames = [0, 128, 255]
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=sig.shape[0],
                   lp_taps=127)
    out = torch.empty((sig.shape[0], len(cfg["dirs"]), cfg["T"]), dtype=torch.float32, device="cuda")
    plan.beamform(torch.from_numpy(sig).cuda(), dm.ENV(dm.KIND_CFDMAS), outs=[out])
    torch.cuda.synchronize()
    env_bench = np.stack([out[f].cpu().numpy() for f in frames])
    del out
    r = plan.beamform(torch.from_numpy(np.ascontiguousarray(sig[frames])).cuda(),
                      dm.RAW(dm.KIND_CFDMAS) | dm.ENV(dm.KIND_CFDMAS))
    torch.cuda.synchronize()
    raw = r[("raw", "cfdmas")].cpu().numpy()
    assert np.array_equal(r[("env", "cfdmas")].cpu().numpy(), env_bench)
    del r
    d = plan.delay_table()
    assert np.array_equal(d, O.delay_table(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"]))
    res = compare_frames(sig, d, 2, {("raw", "cfdmas"): raw, ("env", "cfdmas"): env_bench}, frames)
    assert len(res) == 6
    _assert_whole_frames(res, "C5")


# ------------------------------------------------------------------ edge cases and variants
def test_edge_shapes(dm):
    import torch
    rng = np.random.default_rng(50)
    # T = 1, one direction, n_mics == p
    for (n, p, T, nd) in [(2, 2, 1, 1), (5, 5, 3, 2), (3, 3, 33, 1)]:
        mic = gen.disk_array(n, 0.05, 5e-3, seed=n)
        dirs = gen.az_el_grid(nd, 30.0, 1, 0.0) if nd > 1 else np.array([[0.2, 0.1]])
        sig = rng.standard_normal((2, n, T)).astype(np.float32)
        plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, p, sig, what_all(dm))
        ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, p, sig, env_kinds=KINDS)
        # |E_p| <= C(N,p) max|x| and |A| <= N max|x|: the amplitude scale of every kind
        scale = math.comb(n, p) * float(np.max(np.abs(sig))) + n * float(np.max(np.abs(sig)))
        for key in ref:
            assert_parity(g[key], ref[key], f"edge n={n} p={p} T={T} {key}", zero_scale=scale)
    # n_frames == 0 is a no-op
    plan = dm.Plan(gen.ula(4), gen.az_grid_deg([0, 10]), gen.FS, gen.C_SOUND, 2, 16, max_frames=2)
    res = plan.beamform(torch.zeros((0, 4, 16), device="cuda"), dm.RAW(dm.KIND_DAS))
    assert res[("raw", "das")].shape == (0, 2, 16)
    # all-zero input -> all-zero images (CF guarded by eps)
    res = plan.beamform(torch.zeros((2, 4, 16), device="cuda"), what_all(dm))
    for v in res.values():
        assert float(v.abs().max()) == 0.0
    # too many frames
    with pytest.raises(dm.DmasError):
        plan.beamform(torch.zeros((3, 4, 16), device="cuda"), dm.RAW(dm.KIND_DAS))


def test_short_frames_mostly_out_of_range(dm):
    """T = 16 with delays up to +-65: most gathered samples fall outside [0, T) and read 0."""
    mic = gen.disk_array(32, seed=7)
    dirs = gen.az_el_grid(6, 90.0, 5, 60.0)
    sig = gen.random_signals(2, 32, 16, seed=51)
    plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, 3, sig, what_all(dm))
    assert plan.info["d_max"] > 16
    ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, 3, sig, env_kinds=KINDS)
    for key in ref:
        assert_parity(g[key], ref[key], f"short {key}")


def test_generic_envelope_bandpass_decimation(dm):
    """Generic K4 path: 63-tap low-pass at 8 kHz, a 31-tap band-pass, decimation R = 3; and
    asymmetric band-pass taps (a linear-phase filter tilted by a ramp, and the one-sample delay
    [0, 0, 1]) so that the convolution orientation is fixed on the GPU too."""
    import scipy.signal as ss
    bp = ss.firwin(31, [20e3, 60e3], pass_zero=False, fs=gen.FS).astype(np.float32)
    bp_tilt = (bp * np.linspace(0.3, 1.7, 31)).astype(np.float32)
    delay1 = np.array([0.0, 0.0, 1.0], dtype=np.float32)
    mic = gen.disk_array(16, seed=5)
    dirs = gen.az_el_grid(5, 60.0, 8, 30.0)
    sig = gen.random_signals(2, 16, 1000, seed=52)
    for kw, okw in [(dict(lp_taps=63, lp_cutoff_hz=8000.0, env_decim=3, bp_coeffs=bp),
                     dict(lp_taps=63, cutoff=8000.0, decim=3, bp=bp.astype(np.float64))),
                    (dict(env_decim=4), dict(decim=4)),
                    (dict(bp_coeffs=bp), dict(bp=bp.astype(np.float64))),
                    (dict(bp_coeffs=bp_tilt, env_decim=2), dict(bp=bp_tilt.astype(np.float64), decim=2)),
                    (dict(bp_coeffs=delay1, lp_taps=1), dict(bp=delay1.astype(np.float64), lp_taps=1))]:
        plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, 2, sig, dm.ENV(dm.KIND_DAS | dm.KIND_CFDMAS), **kw)
        ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, 2, sig, kinds=(), env_kinds=("das", "cfdmas"), **okw)
        for key in ref:
            assert_parity(g[key], ref[key], f"generic {kw.keys()} {key}")


def test_cf_eps_zero_nonzero_input(dm):
    mic = gen.disk_array(8, seed=6)
    dirs = gen.az_el_grid(4, 40.0, 4, 20.0)
    sig = gen.random_signals(1, 8, 300, seed=53)
    plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, 2, sig, dm.RAW(dm.KIND_CF | dm.KIND_CFDMAS), cf_eps=0.0)
    ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, 2, sig, kinds=("cf", "cfdmas"), eps=0.0)
    assert_parity(g[("raw", "cf")], ref[("raw", "cf")], "cf eps 0")
    assert float(np.max(g[("raw", "cf")])) <= 1.0 + 1e-5


# ------------------------------------------------------------------ runtime invariances (bitwise)
def test_host_pipeline_matches_device_bitwise(dm):
    import torch
    cfg = gen.config("C5", frames=5)
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"][:2000], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=2)
    what = dm.RAW(dm.KIND_DAS) | dm.ENV(dm.KIND_CFDMAS)
    host = plan.beamform_host(cfg["signals"], what)                # 5 frames through 2-frame stages
    for f0 in range(0, 5, 2):
        x = torch.from_numpy(cfg["signals"][f0:f0 + 2]).cuda()
        dev = plan.beamform(x, what)
        torch.cuda.synchronize()
        for k in dev:
            assert np.array_equal(dev[k].cpu().numpy(), host[k][f0:f0 + 2]), k


def test_chunking_and_sharding_bitwise(dm):
    """Frame chunking (tiny scratch budget -> 1 frame per chunk) and direction sharding (G = 1
    vs 2 / 3 contiguous slices, SPEC.md:323 'bitwise independent of the partitioning') do not
    change a single bit."""
    import torch
    cfg = gen.config("C3")
    sig = np.concatenate([cfg["signals"], gen.random_signals(2, 32, cfg["T"], seed=54)])
    what = dm.RAW(dm.KIND_CFDMAS) | dm.ENV(dm.KIND_CFDMAS | dm.KIND_DAS)
    x = torch.from_numpy(sig).cuda()
    full = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 4, cfg["T"], max_frames=3)
    a = {k: v.cpu().numpy() for k, v in full.beamform(x, what).items()}
    small = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 4, cfg["T"], max_frames=3, scratch_bytes=1)
    b = {k: v.cpu().numpy() for k, v in small.beamform(x, what).items()}
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    nd = len(cfg["dirs"])
    for G in (2, 3):
        bounds = np.linspace(0, nd, G + 1).astype(int)
        for g0, g1 in zip(bounds[:-1], bounds[1:]):
            sh = dm.Plan(cfg["mic_xyz"], cfg["dirs"][g0:g1], cfg["fs"], cfg["c"], 4, cfg["T"], max_frames=3)
            r = sh.beamform(x, what)
            for k in a:
                assert np.array_equal(a[k][:, g0:g1], r[k].cpu().numpy()), (G, k)


def test_calls_on_different_streams_are_ordered(dm):
    """Two calls on one plan issued back to back on two unrelated streams (both use the plan's
    signed-root plane and scratch): the second waits for the first through the plan-owned event,
    so both results equal the sequential ones (cross-stream race)."""
    import torch
    cfg = gen.config("C3")
    sig_a = cfg["signals"]
    sig_b = gen.random_signals(1, 32, cfg["T"], seed=58)
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 3, cfg["T"])
    what = dm.ENV(dm.KIND_CFDMAS) | dm.RAW(dm.KIND_DAS)
    xa, xb = torch.from_numpy(sig_a).cuda(), torch.from_numpy(sig_b).cuda()
    ref_a = {k: v.cpu().numpy() for k, v in plan.beamform(xa, what).items()}
    ref_b = {k: v.cpu().numpy() for k, v in plan.beamform(xb, what).items()}
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs_a = [torch.empty(s, device="cuda") for (_, _, s) in plan.out_shapes(1, what)]
    outs_b = [torch.empty(s, device="cuda") for (_, _, s) in plan.out_shapes(1, what)]
    for _ in range(3):
        plan.beamform(xa, what, outs=outs_a, stream=s1)
        plan.beamform(xb, what, outs=outs_b, stream=s2)
    torch.cuda.synchronize()
    for i, (stage, kind, _) in enumerate(plan.out_shapes(1, what)):
        assert np.array_equal(outs_a[i].cpu().numpy(), ref_a[(stage, kind)]), (stage, kind)
        assert np.array_equal(outs_b[i].cpu().numpy(), ref_b[(stage, kind)]), (stage, kind)


def test_calls_do_not_allocate_and_graph_replay(dm):
    """dmas_beamform allocates nothing (device free memory unchanged across calls, envelope scratch
    included), so a sequence of calls can be captured in a CUDA graph; the replayed images equal
    the eager ones."""
    import torch
    cfg = gen.config("C1")
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=1)
    what = dm.ENV(dm.KIND_CFDMAS | dm.KIND_DAS)
    x = torch.from_numpy(cfg["signals"]).cuda()
    outs = [torch.empty(s, device="cuda") for (_, _, s) in plan.out_shapes(1, what)]
    plan.beamform(x, what, outs=outs)
    torch.cuda.synchronize()
    eager = [o.cpu().numpy() for o in outs]
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        plan.beamform(x, what, outs=outs)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0
    for o in outs:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(4):
                plan.beamform(x, what, outs=outs)
    torch.cuda.synchronize()
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    for o, e in zip(outs, eager):
        assert np.array_equal(o.cpu().numpy(), e)


def test_plans_with_different_windows_coexist(dm):
    """A later plan with a smaller shared-memory window must not break an earlier plan's launches
    (the kernels' dynamic-smem limit is process-wide; dmas_kernels.cu smem_optin)."""
    import torch
    big = dm.Plan(gen.disk_array(64, 0.10, 4e-3, seed=11), gen.az_el_grid(16, 90.0, 16, 60.0), gen.FS,
                  gen.C_SOUND, 3, 2048, max_frames=1)
    xb = torch.from_numpy(gen.random_signals(1, 64, 2048, seed=3)).cuda()
    what = dm.RAW(dm.KIND_ALL) | dm.ENV(dm.KIND_ALL)
    first = {k: v.cpu().numpy() for k, v in big.beamform(xb, what).items()}
    small = dm.Plan(gen.ula(8), gen.az_grid_deg(np.arange(-90, 91, 2)), gen.FS, gen.C_SOUND, 3, 1024, max_frames=1)
    small.beamform(torch.from_numpy(gen.random_signals(1, 8, 1024, seed=4)).cuda(), what)
    again = {k: v.cpu().numpy() for k, v in big.beamform(xb, what).items()}
    torch.cuda.synchronize()
    assert big.n_mics * big.info["window"] > small.n_mics * small.info["window"]
    for k in first:
        assert np.array_equal(first[k], again[k]), k


def test_timing_and_launch_counter(dm):
    import torch
    plan = dm.Plan(gen.ula(8), gen.az_grid_deg(np.arange(-90, 91, 2)), gen.FS, gen.C_SOUND, 2, 1024, max_frames=4)
    x = torch.from_numpy(gen.random_signals(4, 8, 1024, seed=55)).cuda()
    n0 = dm.launch_count()
    plan.set_timing(True)
    plan.beamform(x, dm.ENV(dm.KIND_CFDMAS))
    t = plan.timing_read()
    assert dm.launch_count() - n0 == 3
    assert t["beamform"][1] == 1 and t["envelope"][1] == 1 and t["signed_roots"][1] == 1
    assert all(ms > 0 for ms, c in t.values() if c)


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("T,L", [(4096, 127), (4160, 127), (4132, 127), (8192, 127), (256, 63), (704, 1), (32, 127)])
def test_envelope_engines(dm, engine, T, L):
    """Envelope through the tensor-core low-pass (engine 0: tcgen05 with a 3-pass BF16 split,
    4096-sample tiles, ragged last tile, T % 32 == 0; other T fall back to the FP32 FIR) and the
    FP32 FIR (engine 1), each against the oracle."""
    mic = gen.disk_array(8, 0.05, 5e-3, seed=60)
    dirs = gen.az_el_grid(9, 60.0, 3, 20.0)
    sig = gen.random_signals(2, 8, T, seed=61 + T, sparsity=0.2)
    what = dm.ENV(dm.KIND_CFDMAS | dm.KIND_DAS) | dm.RAW(dm.KIND_DAS)
    plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, 2, sig, what, lp_taps=L, env_engine=engine)
    ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, 2, sig, kinds=("das",), env_kinds=("das", "cfdmas"),
                        lp_taps=L)
    for key in ref:
        assert_parity(g[key], ref[key], f"engine={engine} T={T} L={L} {key}")


def test_envelope_tc_adversarial_split_inputs(dm):
    """The tensor-core envelope's 3-pass BF16 split near its worst case: |y| just below a BF16
    rounding boundary (2^e (1 + 2^-8 - 2^-20): the hi part drops ~2^-8 of the value and the lo part
    carries it), constant rows (every product's error has the same sign), alternating-sign rows
    (|.| must see them as constant), impulses that land on the 34 negative taps, and a wide
    exponent range.  The envelope input is made exact through the slice harness: a 2-microphone
    array at broadside whose second microphone is silent, so DAS = m_0 exactly."""
    import torch
    rng = np.random.default_rng(71)
    T = 4096
    rows = []
    v = 1.0 + 2.0 ** -8 - 2.0 ** -20
    rows.append(np.full(T, v))                                         # constant, worst hi rounding
    rows.append(np.where(np.arange(T) % 2 == 0, v, -v))                # alternating sign
    e = rng.integers(-6, 7, T).astype(np.float64)
    rows.append(np.sign(rng.standard_normal(T)) * np.exp2(e) * v)      # wide exponent range
    imp = np.zeros(T)
    imp[rng.choice(T, 40, replace=False)] = np.exp2(rng.integers(-3, 4, 40)) * v
    rows.append(imp)                                                   # impulses (negative taps)
    steps = np.repeat(np.exp2(rng.integers(-4, 5, T // 64)).astype(np.float64), 64) * v
    rows.append(steps)                                                 # piecewise-constant steps
    sig = np.zeros((len(rows), 2, T), dtype=np.float32)
    sig[:, 0, :] = np.stack(rows).astype(np.float32)
    mic = np.array([[0.0, -0.0015, 0.0], [0.0, 0.0015, 0.0]])
    plan = dm.Plan(mic, [[0.0, 0.0]], gen.FS, gen.C_SOUND, 2, T, max_frames=len(rows))
    res = plan.beamform(torch.from_numpy(sig).cuda(), dm.ENV(dm.KIND_DAS) | dm.RAW(dm.KIND_DAS))
    torch.cuda.synchronize()
    raw = res[("raw", "das")].cpu().numpy()
    assert np.array_equal(raw[:, 0, :], sig[:, 0, :])                 # the envelope input is exact
    env = res[("env", "das")].cpu().numpy()
    h = O.lpf_taps()
    worst = 0.0
    for f in range(len(rows)):
        ref = O.envelope(sig[f, 0, :].astype(np.float64)[None], h)
        err = float(np.max(np.abs(env[f] - ref))) / float(np.max(np.abs(ref)))
        worst = max(worst, err)
        assert_parity(env[f][None], ref[None], f"adversarial envelope row {f}")
    print(f"adversarial envelope worst error {worst:.2e} of peak")
    # the same rows as an envelope-only request: the beamform writes the split plane itself
    env_only = plan.beamform(torch.from_numpy(sig).cuda(), dm.ENV(dm.KIND_DAS))[("env", "das")].cpu().numpy()
    assert np.array_equal(env_only, env)


@pytest.mark.parametrize("p,T,interp", [(2, 4096, 0), (2, 4256, 0), (3, 96, 0), (5, 1056, 0), (2, 2080, 1)])
def test_envelope_presplit_plane(dm, p, T, interp):
    """Envelope-only kinds: the beamform epilogue writes |y| as the BF16 hi / lo split plane and the
    tensor-core envelope reads it with bulk copies (no converter).  Same operands as the converter
    path, so bitwise equal to (a) the raw + envelope request and (b) env_engine = 2 (tensor cores
    on the fp32 image), and within the bar of the oracle.  T covers one tile per row (4096), a
    ragged last tile (4256 = 133 blocks), a row shorter than one tile (96 = 3 blocks: both halo
    edges in one tile) and the interpolating kernel; p = 5 the generic epilogue."""
    import torch
    mic = gen.disk_array(16, 0.08, 5e-3, seed=90 + p)
    dirs = gen.az_el_grid(12, 80.0, 6, 50.0)
    sig = gen.random_signals(2, 16, T, seed=91 + p, sparsity=0.2)
    kinds = dm.KIND_CFDMAS | dm.KIND_DAS | (dm.KIND_CF if p == 5 else 0)
    kw = dict(max_frames=2, delay_interp=interp)
    x = torch.from_numpy(sig).cuda()
    plan = dm.Plan(mic, dirs, gen.FS, gen.C_SOUND, p, T, **kw)
    split = {k: v.cpu().numpy() for k, v in plan.beamform(x, dm.ENV(kinds)).items()}
    both = {k: v.cpu().numpy() for k, v in plan.beamform(x, dm.ENV(kinds) | dm.RAW(kinds)).items()}
    fp32in = dm.Plan(mic, dirs, gen.FS, gen.C_SOUND, p, T, env_engine=2, **kw)
    conv = {k: v.cpu().numpy() for k, v in fp32in.beamform(x, dm.ENV(kinds)).items()}
    torch.cuda.synchronize()
    for key, v in split.items():
        assert np.array_equal(v, both[key]), key
        assert np.array_equal(v, conv[key]), key
    if interp:
        return                           # the interpolating path vs the oracle: test_linear_presteer_parity
    names = [n for n, b in (("das", dm.KIND_DAS), ("cfdmas", dm.KIND_CFDMAS), ("cf", dm.KIND_CF)) if kinds & b]
    ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, p, sig, kinds=(), env_kinds=names)
    for n in names:
        assert_parity(split[("env", n)], ref[("env", n)], f"presplit p={p} T={T} {n}")


# ------------------------------------------------------------------ NEXT-1: matched filter on the GPU
@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_matched_filter_pipeline(dm, name):
    """Raw recordings (T + L - 1 samples, L = 1125-sample chirp) -> GPU matched filter fused with the
    signed roots -> beamform -> envelope, against oracle matched_filter -> beamform_frame -> envelope."""
    cfg = gen.raw_config(name, frames=2)
    p = cfg["order"]
    T = cfg["T"]
    plan, g = run_gpu(dm, cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], p, cfg["signals"],
                      dm.RAW(dm.KIND_DAS | dm.KIND_CFDMAS | dm.KIND_CF) | dm.ENV(dm.KIND_CFDMAS), n_samples=T,
                      mf_coeffs=cfg["chirp"])
    mf = O.matched_filter(cfg["signals"], cfg["chirp"], T)
    ref = oracle_images(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], p, mf, kinds=("das", "cfdmas", "cf"),
                        env_kinds=("cfdmas",))
    for key in ref:
        assert_parity(g[key], ref[key], f"MF {name} {key}")


def test_matched_filter_host_path_and_validation(dm):
    import torch
    cfg = gen.raw_config("C1", frames=3)
    plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=2,
                   mf_coeffs=cfg["chirp"])
    what = dm.ENV(dm.KIND_CFDMAS)
    host = plan.beamform_host(cfg["signals"], what)
    dev = plan.beamform(torch.from_numpy(cfg["signals"][:2]).cuda(), what)
    assert np.array_equal(dev[("env", "cfdmas")].cpu().numpy(), host[("env", "cfdmas")][:2])
    with pytest.raises(ValueError):                                   # matched-filtered length is rejected
        plan.beamform(torch.zeros((1, 8, cfg["T"]), device="cuda"), what)
    with pytest.raises(dm.DmasError):
        dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], mf_coeffs=np.zeros(16))


# ------------------------------------------------------------------ NEXT-3: orders 6..8 (general partition formula)
@pytest.mark.parametrize("p", [6, 7, 8])
def test_high_orders_config_C3(dm, p):
    """Orders 6..8 through the general Newton-Girard partition formula on the C3
    scene (32 mics >= 2p), every kind raw + envelope, against the oracle's Vieta E_p."""
    cfg = gen.config("C3")
    dirs = cfg["dirs"][::3]
    plan, g = run_gpu(dm, cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], p, cfg["signals"], what_all(dm))
    ref = oracle_images(cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], p, cfg["signals"], env_kinds=KINDS)
    for key in ref:
        assert_parity(g[key], ref[key], f"C3 p={p} {key}")


@pytest.mark.parametrize("p", [6, 7, 8])
def test_high_orders_slice_bruteforce(dm, p):
    """Broadside slice harness: random slices of N = 2p microphones against Eq. (5) brute force."""
    import torch
    rng = np.random.default_rng(80 + p)
    n, T = 2 * p, 200
    x = rng.uniform(-1, 1, (n, T)).astype(np.float32)
    plan = _slice_plan(dm, n, p, T)
    g = plan.beamform(torch.from_numpy(x[None]).cuda(), dm.RAW(dm.KIND_DMAS))[("raw", "dmas")].cpu().numpy()[0, 0]
    ref = np.array([O.brute_force_esp(list(O.signed_root(x[:, t].astype(np.float64), p)), p) for t in range(T)])
    assert np.max(np.abs(g - ref)) <= TOL * np.max(np.abs(ref))


# ------------------------------------------------------------------ NEXT-2: linear-interpolation pre-steering
@pytest.mark.parametrize("name,p", [("C1", 2), ("C2", 2), ("C3", 3), ("C3", 5)])
def test_linear_presteer_parity(dm, name, p):
    """delay_interp = 1: floor table bit-exact, fractions to fp32 rounding, every kind raw + envelope
    against the oracle's gather_linear -> beamform_frame."""
    cfg = gen.config(name)
    dirs = cfg["dirs"] if name == "C1" else cfg["dirs"][::2]
    plan, g = run_gpu(dm, cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], p, cfg["signals"], what_all(dm), delay_interp=1)
    d0, al = O.delay_table(cfg["mic_xyz"], dirs, cfg["fs"], cfg["c"], mode="linear")
    assert np.array_equal(plan.delay_table(), d0)
    assert np.max(np.abs(plan.delay_fraction() - al)) <= 6e-8
    ref = {}
    h = O.lpf_taps()
    img = O.beamform_frame(cfg["signals"][0], d0, p, alpha=al)
    for k in KINDS:
        ref[("raw", k)] = img[k][None]
        ref[("env", k)] = O.envelope(img[k], h)[None]
    for key in ref:
        assert_parity(g[key], ref[key], f"linear {name} p={p} {key}")


def test_linear_presteer_with_matched_filter_and_slices(dm):
    """Linear pre-steering composed with the GPU matched filter; and the broadside slice harness
    (all fractions 0) reproduces the integer path's brute-force values."""
    import torch
    cfg = gen.raw_config("C1", frames=1)
    plan, g = run_gpu(dm, cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["signals"],
                      dm.RAW(dm.KIND_CFDMAS) | dm.ENV(dm.KIND_CFDMAS), n_samples=cfg["T"], mf_coeffs=cfg["chirp"],
                      delay_interp=1)
    mf = O.matched_filter(cfg["signals"][0], cfg["chirp"], cfg["T"])
    d0, al = O.delay_table(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], mode="linear")
    img = O.beamform_frame(mf, d0, 2, alpha=al)
    assert_parity(g[("raw", "cfdmas")], img["cfdmas"][None], "MF+linear raw")
    assert_parity(g[("env", "cfdmas")], O.envelope(img["cfdmas"], O.lpf_taps())[None], "MF+linear env")
    x = np.random.default_rng(91).uniform(-1, 1, (7, 64)).astype(np.float32)
    mic = np.stack([np.zeros(7), 0.003 * np.arange(7), np.zeros(7)], axis=1)
    plan = dm.Plan(mic, [[0.0, 0.0]], gen.FS, gen.C_SOUND, 3, 64, delay_interp=1)
    assert np.all(plan.delay_fraction() == 0)
    r = plan.beamform(torch.from_numpy(x[None]).cuda(), dm.RAW(dm.KIND_DMAS))[("raw", "dmas")].cpu().numpy()[0, 0]
    ref = np.array([O.brute_force_esp(list(O.signed_root(x[:, t].astype(np.float64), 3)), 3) for t in range(64)])
    assert np.max(np.abs(r - ref)) <= 1e-5 * np.max(np.abs(ref))


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("what_name", ["env_all", "raw_env_mix"])
def test_sharded_plan_one_rank_bitwise(dm, what_name, fused):
    """A one-rank sharded plan (n_ranks = 1 with an NCCL comm id: the exchange code runs on one GPU --
    the communicator, the in-place ncclBroadcast per chunk, the comm-stream ordering, the gather
    staging and the gather schedule's local copies) returns images bitwise equal to a plain plan's:
    resident shards, images gathered onto the root over several double-buffered exchange chunks,
    and the host-buffer path ("G = 1 vs G > 1 bitwise"; the G > 1 exchange is
    checked on the CPU by tests/test_parallel.py::test_gather_schedule_assembles_the_image)."""
    import torch
    cfg = gen.config("C3")
    sig = np.concatenate([cfg["signals"], gen.random_signals(4, 32, cfg["T"], seed=56)])   # 5 frames
    x = torch.from_numpy(sig).cuda()
    what = dm.ENV(dm.KIND_ALL) if what_name == "env_all" else dm.RAW(dm.KIND_CFDMAS) | dm.ENV(dm.KIND_CFDMAS | dm.KIND_DAS)
    args = (cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 3, cfg["T"])
    plain = dm.Plan(*args, max_frames=5, scratch_bytes=1)       # 1 frame per chunk (5 envelope-only kinds)
    ref = {k: v.cpu().numpy() for k, v in plain.beamform(x, what).items()}
    sp = dm.Plan(*args, max_frames=5, scratch_bytes=1, n_ranks=1, rank=0, root=0, comm_id=dm.comm_id(),
                 fused_gather=fused)
    assert sp.sharded and sp.info["n_dirs_total"] == len(cfg["dirs"]) and sp.info["dir_begin"] == 0
    assert np.array_equal(sp.delay_table(), plain.delay_table())
    resident = sp.beamform(x.clone(), what)
    gathered = sp.beamform(x.clone(), what | dm.GATHER)
    host = sp.beamform_host(sig, what)                      # every rank's shard into its host buffers
    host_g = sp.beamform_host(sig, what | dm.GATHER)        # gathered onto the root, then to the host
    torch.cuda.synchronize()
    for k in ref:
        assert np.array_equal(resident[k].cpu().numpy(), ref[k]), ("resident", k)
        assert np.array_equal(gathered[k].cpu().numpy(), ref[k]), ("gathered", k)
        assert np.array_equal(host[k], ref[k]), ("host", k)
        assert np.array_equal(host_g[k], ref[k]), ("host gathered", k)
    sp.close()


# ------------------------------------------------------------------ large arrays (microphone-group path)
@pytest.mark.parametrize("kind", ["disk160", "hex3cm", "hex6cm"])
def test_large_array_parity(dm, kind):
    """Arrays too large for one shared-memory window (e.g. the 5 mm hexagonal lattices of
    PAPER.md:243-247) stream microphone groups through the TMA window; same arithmetic."""
    if kind == "disk160":
        mic, p, T = gen.disk_array(160, 0.10, 3.5e-3, seed=12), 2, 700
    elif kind == "hex3cm":
        mic, p, T = gen.hex_array(0.03), 3, 512
    else:
        mic, p, T = gen.hex_array(0.06), 2, 512
    dirs = gen.az_el_grid(9, 80.0, 2, 10.0)
    sig = gen.random_signals(2, len(mic), T, seed=len(mic), sparsity=0.1)
    plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, p, sig, what_all(dm))
    assert plan.info["psi_tile"] == 8            # the microphone-group path was taken
    ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, p, sig, env_kinds=KINDS)
    for key in ref:
        assert_parity(g[key], ref[key], f"{kind} {key}")
    # and with linear pre-steering
    plan, g = run_gpu(dm, mic, dirs, gen.FS, gen.C_SOUND, p, sig[:1], dm.RAW(dm.KIND_CFDMAS), delay_interp=1)
    d0, al = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND, mode="linear")
    assert_parity(g[("raw", "cfdmas")], O.beamform_frame(sig[0], d0, p, alpha=al)["cfdmas"][None], f"{kind} linear")


def test_beamform_kernel_for_benchmark_configs(dm):
    """All three take the LDS.64 kernel: C5 with 256-sample tiles of 64 k-d-grouped directions; C2
    with 32-direction k-d tiles (its consecutive rows straddle its 30-direction elevation columns);
    C4 (64 mics) with 128-sample tiles of 64 k-d-grouped directions (4 pixels per lane: the
    256-sample windows of 64 microphones would not fit 2 CTAs per SM).  bf_engine = 1 forces the
    classic kernel."""
    for name, k, order, tt, psi in (("C2", 1, 1, 256, 32), ("C4", 1, 1, 128, 64), ("C5", 1, 1, 256, 64)):
        cfg = gen.config(name, frames=1)
        plan = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], cfg["order"], cfg["T"])
        assert plan.info["psi_tile"] == psi and plan.info["bf_kernel"] == k, (name, plan.info)
        assert plan.info["tile_order"] == order and plan.info["t_tile"] == tt, (name, plan.info)
        classic = dm.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], cfg["order"], cfg["T"], bf_engine=1)
        assert classic.info["bf_kernel"] == 0


# ------------------------------------------------------------------ LDS.64 kernel (k_beamform_lds64)
@pytest.mark.parametrize("case", ["C5p2", "C5p3", "C5p4", "C5p5", "C2p2", "C4p3", "C4p5", "ragged", "ragged_p6", "tiny",
                                  "short_T", "scattered", "kt4_ragged", "C5p2i", "C5p3i", "C5p5i", "C2p2i",
                                  "ragged_i"])
def test_lds64_kernel_bitwise_and_parity(dm, case):
    """k_beamform_lds64 (paired root plane, one LDS.64 per 2 pixels, pixel-pair packed FP32)
    performs the same per-pixel operations in the same microphone order as the classic kernel:
    images are bit-identical across ragged direction tiles (n_dirs % 32 != 0), ragged sample tiles
    (T % 256 != 0), T shorter than the delay spread, every kind, orders 2..6; and within the
    north_star bar of the oracle."""
    import torch
    what = what_all(dm)
    interp = case.endswith("i")                               # linear pre-steering (NEXT-2)
    case = case[:-1] if interp else case
    if case.startswith("C5"):                               # C5's array, scene and grid: 300 directions
        cfg = gen.config("C5", frames=2)                      # (9 full 32-direction tiles + 12), T = 4096
        p = int(case[-1])
        mic, dirs, sig = cfg["mic_xyz"], cfg["dirs"][:300], cfg["signals"]
    elif case.startswith("C4"):                             # 64 mics: 4 pixels per lane, k-d tiles
        cfg = gen.config("C4", frames=1)
        p, mic, dirs, sig = int(case[-1]), cfg["mic_xyz"], cfg["dirs"][:300], cfg["signals"]
    elif case == "kt4_ragged":                               # 64 mics: 4 pixels per lane, T = 301
        p, mic = 2, gen.disk_array(64, 0.10, 4e-3, seed=11)   # (2 full 128-sample tiles + 45),
        dirs = gen.az_el_grid(10, 20.0, 10, 10.0)             # 100 directions (3 full 32-tiles + 4)
        sig = gen.random_signals(2, 64, 301, seed=67, sparsity=0.1)
    elif case == "scattered":                                # 500 random directions in random order:
        cfg = gen.config("C5", frames=1)                      # only k-d tiles can fit the window
        rng = np.random.default_rng(66)
        dirs = np.stack([rng.uniform(-1.2, 1.2, 500), rng.uniform(-0.9, 0.9, 500)], axis=1)
        p, mic, sig = 2, cfg["mic_xyz"], cfg["signals"][:, :, :1024].copy()
    elif case == "C2p2":                                     # k-d tiles (rows scattered by psi_map)
        cfg = gen.config("C2")
        p, mic, dirs, sig = 2, cfg["mic_xyz"], cfg["dirs"], cfg["signals"]
    elif case.startswith("ragged"):
        p = 6 if case.endswith("p6") else 2 if not interp else 3
        mic = gen.disk_array(24 if p == 6 else 13, 0.09, 5e-3, seed=61)
        dirs = gen.az_el_grid(23, 85.0, 7, 55.0)            # 161 directions: 5 full tiles + 1
        sig = gen.random_signals(2, len(mic), 601, seed=62, sparsity=0.2)   # 2 full 256-tiles + 89
    elif case == "tiny":
        p, mic, dirs = 3, gen.disk_array(5, 0.05, 5e-3, seed=63), gen.az_el_grid(3, 40.0, 1, 0.0)
        sig = gen.random_signals(1, 5, 3, seed=64)
    else:                                                    # T = 40 < delay spread (+-65)
        p, mic, dirs = 2, gen.disk_array(32, seed=7), gen.az_el_grid(3, 30.0, 32, 10.0)
        sig = gen.random_signals(2, 32, 40, seed=65, sparsity=0.1)
    x = torch.from_numpy(np.ascontiguousarray(sig)).cuda()
    res = []
    for eng in (0, 1):
        plan = dm.Plan(mic, dirs, gen.FS, gen.C_SOUND, p, sig.shape[2], max_frames=sig.shape[0], bf_engine=eng,
                       delay_interp=1 if interp else 0)
        assert plan.info["bf_kernel"] == (1 if eng == 0 else 0), plan.info
        if case == "scattered" and eng == 0:
            assert plan.info["tile_order"] == 1, plan.info
        if case == "kt4_ragged" and eng == 0:
            assert plan.info["t_tile"] == 128, plan.info
        r = plan.beamform(x, what)
        torch.cuda.synchronize()
        res.append({k: v.cpu().numpy() for k, v in r.items()})
    for k in res[1]:
        assert np.array_equal(res[0][k], res[1][k]), (case, interp, k)
    if interp:
        d0, al = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND, mode="linear")
        ref = {}
        h = O.lpf_taps()
        for f in range(sig.shape[0]):
            img = O.beamform_frame(sig[f], d0, p, alpha=al)
            for k in KINDS:
                ref.setdefault(("raw", k), []).append(img[k])
                ref.setdefault(("env", k), []).append(O.envelope(img[k], h))
        ref = {k: np.stack(v) for k, v in ref.items()}
    else:
        ref = oracle_images(mic, dirs, gen.FS, gen.C_SOUND, p, sig, env_kinds=KINDS)
    scale = math.comb(len(mic), p) * float(np.max(np.abs(sig))) + len(mic) * float(np.max(np.abs(sig)))
    for key in ref:
        assert_parity(res[0][key], ref[key], f"lds64 {case} {key}", zero_scale=scale)


@pytest.mark.parametrize("case", ["C5", "kt4", "ragged", "raw_mf"])
def test_das_only_identity_plane(dm, case):
    """A DAS-only request (raw and/or envelope) on the LDS.64 path sums the samples themselves
    (identity plane, one FADD2 per pixel pair) instead of rebuilding x from the signed roots:
    within the oracle bar, and within fp32 rounding of the DAS an all-kinds request returns."""
    import torch
    kw = {}
    if case == "C5":
        cfg = gen.config("C5", frames=2)
        mic, dirs, sig, T = cfg["mic_xyz"], cfg["dirs"][:300], cfg["signals"], cfg["T"]
    elif case == "kt4":
        mic, dirs = gen.disk_array(64, 0.10, 4e-3, seed=11), gen.az_el_grid(10, 20.0, 10, 10.0)
        sig = gen.random_signals(2, 64, 301, seed=68, sparsity=0.1)
        T = 301
    elif case == "ragged":
        mic, dirs = gen.disk_array(13, 0.09, 5e-3, seed=61), gen.az_el_grid(23, 85.0, 7, 55.0)
        sig = gen.random_signals(2, 13, 601, seed=69, sparsity=0.2)
        T = 601
    else:
        cfg = gen.raw_config("C1", frames=2)
        mic, dirs, T = cfg["mic_xyz"], cfg["dirs"], cfg["T"]
        kw["mf_coeffs"] = cfg["chirp"]
        sig = cfg["signals"]
    plan = dm.Plan(mic, dirs, gen.FS, gen.C_SOUND, 3, T, max_frames=sig.shape[0], **kw)
    assert plan.info["bf_kernel"] == 1, plan.info
    if case == "kt4":
        assert plan.info["t_tile"] == 128, plan.info          # the 4-pixel-per-lane DAS variant ran
    x = torch.from_numpy(np.ascontiguousarray(sig)).cuda()
    das = plan.beamform(x, dm.RAW(dm.KIND_DAS) | dm.ENV(dm.KIND_DAS))
    env_only = plan.beamform(x, dm.ENV(dm.KIND_DAS))[("env", "das")].cpu().numpy()
    full = plan.beamform(x, what_all(dm))
    torch.cuda.synchronize()
    g_raw, g_env = das[("raw", "das")].cpu().numpy(), das[("env", "das")].cpu().numpy()
    assert np.array_equal(g_env, env_only)
    m = O.matched_filter(sig, cfg["chirp"], T) if case == "raw_mf" else sig
    d = O.delay_table(mic, dirs, gen.FS, gen.C_SOUND)
    h = O.lpf_taps()
    for f in range(sig.shape[0]):
        ref = O.beamform_frame(m[f], d, 3)["das"]
        assert_parity(g_raw[f][None], ref[None], f"das-only {case} raw f{f}")
        assert_parity(g_env[f][None], O.envelope(ref, h)[None], f"das-only {case} env f{f}")
        fr = full[("raw", "das")][f].cpu().numpy()
        assert np.max(np.abs(fr - g_raw[f])) <= 1e-5 * np.max(np.abs(fr))
