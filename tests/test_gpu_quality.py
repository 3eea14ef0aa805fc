"""NEXT-4: the paper's §III-A image-quality trends, measured through the GPU path
(experiments/quality.py), and the same figures of merit computed from the float64 oracle.

Trends asserted (PAPER.md citations):
* :65, :123, :201  — DMAS raises the PSF dynamic range over DAS; higher order raises it further;
                     CF raises it again.
* :203              — no discernible change in range resolution across beamformers.
* :185, :231-236    — image SNR rises with order and with CF (for input SNR well above the
                     noise floor).
* :243-249          — beamwidth falls as the array grows, for every beamformer.

The paper's absolute numbers depend on definitions it does not give (reading Q20), so
the GPU values are checked against the oracle's on the same scene, not against printed numbers.
"""

import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "experiments"))

import quality  # noqa: E402

import oracle  # noqa: E402
from workloads import gen  # noqa: E402


def oracle_beamform(mic, dirs, sig, p, kinds):
    """Same contract as quality._beamform, from the float64 oracle (test infrastructure)."""
    d = oracle.delay_table(mic, dirs, gen.FS, gen.C_SOUND)
    img = oracle.beamform_frame(sig.astype(np.float64), d, p)
    taps = oracle.lpf_taps(127, 5000.0, gen.FS)
    return {k: oracle.envelope(img[k], taps) for k in kinds}


def _metrics_consistent(psf):
    for name in ("DAS", "DMAS2", "DMAS3", "DMAS4", "DMAS5"):
        assert abs(psf[name]["peak_az_deg"] - 10.0) <= 1.0, (name, psf[name])


def _assert_psf_trends(psf):
    _metrics_consistent(psf)
    dr = {k: v["dynamic_range_db"] for k, v in psf.items()}
    assert dr["DMAS2"] > dr["DAS"] + 3.0, dr
    for a, b in (("DMAS2", "DMAS3"), ("DMAS3", "DMAS4"), ("DMAS4", "DMAS5")):
        assert dr[b] > dr[a], (a, b, dr)
    for k in ("DAS", "DMAS2", "DMAS3", "DMAS4", "DMAS5"):
        assert dr[k + "-CF"] > dr[k], (k, dr)
    widths = [v["range_width_samples"] for v in psf.values()]
    assert max(widths) <= 1.25 * min(widths), widths


def test_psf_metrics_on_oracle():
    """The figure-of-merit code on the oracle's images (CPU): the paper's PSF trends hold."""
    psf = quality.psf_sweep(beamform=oracle_beamform)
    _assert_psf_trends(psf)
    assert psf["DMAS5-CF"]["dynamic_range_db"] > 75.0        # PAPER.md:123 "almost 80 dB"


def test_beamwidth_metric_closed_form():
    """beamwidth_deg on a sampled Gaussian profile recovers its analytic -3 dB width."""
    az = np.arange(-30.0, 30.01, 0.25)
    sigma = 4.0
    prof = np.exp(-az ** 2 / (2 * sigma ** 2))
    w = quality.beamwidth_deg(np.stack([prof, prof * 0.5], axis=1), az)
    assert w == pytest.approx(2 * sigma * math.sqrt(math.log(2.0)), rel=2e-3)


@pytest.mark.gpu
def test_psf_trends_gpu_match_oracle():
    gpu = quality.psf_sweep()
    _assert_psf_trends(gpu)
    ref = quality.psf_sweep(beamform=oracle_beamform)
    for k in gpu:
        print(k, gpu[k]["dynamic_range_db"], ref[k]["dynamic_range_db"])
        assert gpu[k]["peak_az_deg"] == ref[k]["peak_az_deg"], k
        assert gpu[k]["range_width_samples"] == ref[k]["range_width_samples"], k
        # side lobes sit 13-79 dB below the peak; fp32 accumulation and the BF16-split envelope
        # are relative-accurate to ~1e-5 there, i.e. well under 0.5 dB
        assert gpu[k]["dynamic_range_db"] == pytest.approx(ref[k]["dynamic_range_db"], abs=0.5), k
    assert ref["DMAS5-CF"]["dynamic_range_db"] > 75.0       # PAPER.md:123 "almost 80 dB"


@pytest.mark.gpu
def test_image_snr_trends_gpu():
    res = quality.image_snr_sweep(snrs=(-10.0, 10.0), seeds=(1, 2))
    for snr, row in res.items():
        for k in ("DAS", "DMAS2", "DMAS3", "DMAS4", "DMAS5"):
            assert row[k + "-CF"] > row[k], (snr, k, row)
        assert row["DMAS3"] > row["DAS"], (snr, row)
    hi = res["10.0"]
    assert hi["DMAS2"] > hi["DAS"] and hi["DMAS5"] > hi["DMAS3"], hi
    # more input SNR never makes the image worse
    for k in res["10.0"]:
        assert res["10.0"][k] > res["-10.0"][k] - 0.5, k


@pytest.mark.gpu
def test_beamwidth_falls_with_radius_gpu():
    res = quality.beamwidth_sweep(radii=(0.01, 0.03, 0.06))
    rows = [res[k] for k in ("1cm", "3cm", "6cm")]
    for k in ("DAS", "DMAS2", "DMAS3", "DMAS5", "DMAS5-CF"):
        assert rows[0][k] > rows[1][k] > rows[2][k], (k, rows)
    for r in rows:                                # DMAS narrows the main lobe relative to DAS
        assert r["DMAS3"] < r["DAS"], r
    spread = [max(v for k, v in r.items() if k != "n_mics") - min(v for k, v in r.items() if k != "n_mics")
              for r in rows]
    assert spread[0] > spread[1] > spread[2], spread   # PAPER.md:243 beamwidths converge


def test_image_snr_metric_hand_computed():
    """E_off / image SNR (reading Q20) on a hand-built image: peak 8 at the target
    (az 0, t 2000); every pixel inside the guard (|az| <= 15 deg AND |t - 2000| <= 1125) is 4 and
    must be ignored; the 76 rows outside +-15 deg are 0.5 (76 x 4000 pixels) and the 15 rows inside
    it are 0.25 outside the range guard (15 x 1749 pixels), so after normalising to the peak
    E_off = (76*4000*0.5 + 15*1749*0.25) / (76*4000 + 15*1749) / 8 and SNR = 20 log10(1 / E_off)."""
    az = np.arange(-90.0, 91.0, 2.0)
    T = 4000
    t = np.arange(T)
    in_az = np.abs(az) <= 15.0
    assert in_az.sum() == 15 and (~in_az).sum() == 76
    env = np.where(in_az[:, None], 0.25, 0.5) * np.ones((1, T))
    guard = in_az[:, None] & (np.abs(t - 2000)[None, :] <= 1125)
    assert guard.sum() == 15 * 2251
    env[guard] = 4.0
    env[np.argmin(np.abs(az)), 2000] = 8.0
    e_off = (76 * 4000 * 0.5 + 15 * 1749 * 0.25) / (76 * 4000 + 15 * 1749) / 8.0
    assert quality.image_snr(env, az, 0.0, 2000) == pytest.approx(20 * math.log10(1.0 / e_off), abs=1e-12)
    # and the guard really matters: without it the 4.0 plateau raises E_off
    assert quality.image_snr(env, az, 0.0, 2000, guard_deg=-1.0) < 20 * math.log10(1.0 / e_off) - 1.0


@pytest.mark.gpu
def test_image_snr_gpu_matches_oracle():
    """Fig. 3 sweep: image SNR of every beamformer, with and without CF, at two
    input SNRs -- GPU envelope images against the float64 oracle's on the same noisy scenes."""
    gpu = quality.image_snr_sweep(snrs=(-10.0, 10.0), seeds=(1,))
    ref = quality.image_snr_sweep(beamform=oracle_beamform, snrs=(-10.0, 10.0), seeds=(1,))
    for snr in gpu:
        for k in gpu[snr]:
            assert gpu[snr][k] == pytest.approx(ref[snr][k], abs=0.01), (snr, k, gpu[snr][k], ref[snr][k])


@pytest.mark.gpu
def test_beamwidth_gpu_matches_oracle():
    """Fig. 6 sweep: -3 dB beamwidth on 5 mm hexagonal lattices of radius 1 and
    2 cm, every beamformer with and without CF -- GPU against the oracle's images."""
    gpu = quality.beamwidth_sweep(radii=(0.01, 0.02))
    ref = quality.beamwidth_sweep(beamform=oracle_beamform, radii=(0.01, 0.02))
    for r in gpu:
        assert gpu[r]["n_mics"] == ref[r]["n_mics"]
        for k, v in gpu[r].items():
            assert v == pytest.approx(ref[r][k], abs=1e-3), (r, k, v, ref[r][k])
