"""C-ABI library checks that need no GPU: the .so builds/loads, exports every symbol that
include/dmas.h declares, and its host-side validation rejects bad descriptors before any
device work (the codes of include/dmas.h)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dmas.h")


@pytest.fixture(scope="module")
def dm():
    from paper_2511_09165_b200 import _build
    _build.build()
    from paper_2511_09165_b200 import dmas
    return dmas


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dmas_[a-z_]+)\s*\(", src)) - {"dmas_plan_t"})


def test_header_declares_expected_calls():
    names = header_functions()
    for n in ("dmas_plan", "dmas_beamform", "dmas_destroy", "dmas_delay_table", "dmas_beamform_host"):
        assert n in names


def test_so_exports_every_header_symbol(dm):
    out = subprocess.run(["nm", "-D", "--defined-only", dm._LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dmas_\w+)", out))
    missing = [n for n in header_functions() if n not in exported]
    assert not missing, missing
    assert set(dm.EXPORTS) == set(header_functions())


def test_header_compiles_as_c():
    src = '#include "dmas.h"\nint main(void){dmas_plan_desc d; dmas_plan_desc_init(&d); return d.order == 2 ? 0 : 1;}\n'
    tmp = "/tmp/_dmas_hdr_test.c"
    open(tmp, "w").write(src)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), tmp],
                   check=True)


def test_desc_defaults(dm):
    d = dm.dmas_plan_desc()
    dm.lib.dmas_plan_desc_init(ctypes.byref(d))
    assert (d.order, d.lp_taps, d.lp_cutoff_hz, d.env_decim, d.device, d.max_frames) == (2, 127, 5000.0, 1, -1, 1)
    assert d.cf_eps == pytest.approx(1e-30, rel=1e-6)


def test_status_strings(dm):
    for code, name in dm.STATUS.items():
        assert dm.lib.dmas_status_string(code).decode() == name


def _plan_err(dm, **kw):
    base = dict(mic_xyz=np.array([[0, 0.01, 0], [0, -0.01, 0], [0, 0, 0.01]]), dir_az_el=np.zeros((4, 2)),
                fs=450e3, c=343.0, order=2, n_samples=64)
    base.update(kw)
    args = [base.pop(k) for k in ("mic_xyz", "dir_az_el", "fs", "c", "order", "n_samples")]
    with pytest.raises(dm.DmasError) as ei:
        dm.Plan(*args, **base)
    return ei.value.status


def test_validation_errors(dm):
    """Host-side validation (include/dmas.h DMAS_ERR_*) happens before any CUDA call."""
    assert _plan_err(dm, order=9) == 3
    assert _plan_err(dm, order=1) == 3
    twelve = np.stack([np.zeros(11), 0.004 * np.arange(11), np.zeros(11)], axis=1)
    assert _plan_err(dm, order=6, mic_xyz=twelve) == 3     # p >= 6 needs n_mics >= 2p
    assert _plan_err(dm, order=4) == 3                      # n_mics (3) < p  (SPEC "N < n")
    assert _plan_err(dm, c=0.0) == 2
    assert _plan_err(dm, fs=-1.0) == 2
    assert _plan_err(dm, n_samples=0) == 2
    assert _plan_err(dm, lp_taps=126) == 2
    assert _plan_err(dm, lp_cutoff_hz=300e3) == 2
    assert _plan_err(dm, env_decim=0) == 2
    assert _plan_err(dm, cf_eps=-1.0) == 2
    assert _plan_err(dm, max_frames=0) == 2
    assert _plan_err(dm, mic_xyz=np.array([[0, 0.01, 0], [0, 0.01, 0], [0, 0, 0.02]])) == 2   # duplicate
    assert _plan_err(dm, mic_xyz=np.array([[0, np.nan, 0], [0, 0.01, 0], [0, 0, 0.02]])) == 2
    assert _plan_err(dm, dir_az_el=np.array([[4.0, 0.0]])) == 2                             # theta > pi
    assert _plan_err(dm, dir_az_el=np.array([[0.0, 1.6]])) == 2                             # phi > pi/2
    assert _plan_err(dm, bp_coeffs=[1.0, 2.0]) == 2                                         # even bp length
    assert _plan_err(dm, mf_coeffs=np.zeros(8)) == 2                                        # zero-energy chirp
    assert _plan_err(dm, mf_coeffs=np.ones(20000)) == 2                                     # too many taps
    assert _plan_err(dm, mf_coeffs=np.array([1.0, np.inf])) == 2
    assert _plan_err(dm, bf_engine=2) == 2
    assert _plan_err(dm, env_engine=3) == 2
    assert _plan_err(dm, delay_interp=2) == 2


def test_struct_layouts_match_header(dm):
    """The ctypes mirrors of dmas_plan_desc / dmas_plan_info have the C compiler's layout: field
    offsets and sizes from a tiny C program built against include/dmas.h."""
    fields = {"dmas_plan_desc": dm.dmas_plan_desc, "dmas_plan_info": dm.dmas_plan_info}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "dmas.h"', 'int main(void){']
    for sname, cls in fields.items():
        src.append(f'printf("{sname} sizeof %zu\\n", sizeof({sname}));')
        for fname, _ in cls._fields_:
            src.append(f'printf("{sname} {fname} %zu\\n", offsetof({sname}, {fname}));')
    src.append("return 0;}")
    c, exe = "/tmp/_dmas_layout.c", "/tmp/_dmas_layout"
    open(c, "w").write("\n".join(src) + "\n")
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for sname, cls in fields.items():
        assert got[(sname, "sizeof")] == ctypes.sizeof(cls), sname
        for fname, _ in cls._fields_:
            assert got[(sname, fname)] == getattr(cls, fname).offset, (sname, fname)


def test_null_handling(dm):
    assert dm.lib.dmas_plan(None, None) == 1
    h = ctypes.c_void_p()
    assert dm.lib.dmas_plan(None, ctypes.byref(h)) == 1
    assert not h.value
    dm.lib.dmas_destroy(None)                               # NULL-safe
    assert dm.lib.dmas_delay_table(None, None) == 1
    assert dm.lib.dmas_beamform(None, None, 0, None, 1, None) == 1
    assert isinstance(dm.launch_count(), int)
