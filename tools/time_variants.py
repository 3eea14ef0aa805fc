#!/usr/bin/env python
"""Time library variants (tools/build_variants.sh) on the C5 step's launch and check that they
return bitwise the same images (experiments; each variant runs in its own process through
DMAS_LIBRARY).

usage: python tools/time_variants.py build/libdmas_A.so build/libdmas_B.so ...   (on a GPU box)
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, sys, time
sys.path.insert(0, ROOT)
import numpy as np, torch
from workloads import gen
from paper_2511_09165_b200 import dmas
F = 16
cfg = gen.config("C5", frames=F)
x = torch.from_numpy(cfg["signals"]).cuda()
import os
KW = json.loads(os.environ.get("DMAS_TV_KW", "{}"))      # extra plan options, e.g. {"delay_interp": 1}
plan = dmas.Plan(cfg["mic_xyz"], cfg["dirs"], cfg["fs"], cfg["c"], 2, cfg["T"], max_frames=F, **KW)
out = torch.empty((F, len(cfg["dirs"]), cfg["T"]), dtype=torch.float32, device="cuda")
what = dmas.ENV(dmas.KIND_CFDMAS)
for _ in range(3):
    plan.beamform(x, what, outs=[out])
torch.cuda.synchronize()
plan.set_timing(True)
for _ in range(REPS):
    plan.beamform(x, what, outs=[out])
torch.cuda.synchronize()
t = plan.timing_read()
h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
rec = {"lib": LIB, "env_ms": t["envelope"][0] / t["envelope"][1], "bf_ms": t["beamform"][0] / t["beamform"][1], "sha": h}
from oracle import dmas_oracle as O                 # sanity: 128 rows of frame 0 against the oracle
rows = np.linspace(0, len(cfg["dirs"]) - 1, 128).astype(int)
if KW.get("delay_interp"):
    d, al = O.delay_table(cfg["mic_xyz"], cfg["dirs"][rows], cfg["fs"], cfg["c"], mode="linear")
else:
    d, al = O.delay_table(cfg["mic_xyz"], cfg["dirs"][rows], cfg["fs"], cfg["c"]), None
ref = O.envelope(O.beamform_frame(cfg["signals"][0], d, 2, alpha=al)["cfdmas"], O.lpf_taps())
got = out[0].cpu().numpy()[rows]
rec["oracle_rel_err"] = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
try:                                     # role-wait profile (builds with -DDMAS_TC_PROFILE)
    import ctypes
    fn = dmas.lib.dmas_tc_prof_read
    buf = (ctypes.c_ulonglong * (148 * 12))()
    if fn(buf) == 0:
        a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 6, 2).astype(np.float64)
        tot = a[:, 5, 0]
        names = ["tma", "mma", "conv", "epi", "copy"]
        rec["wait_frac"] = {names[r]: [float(np.mean(a[:, r, 0] / tot)), float(np.mean(a[:, r, 1] / tot))]
                            for r in range(5)}
except AttributeError:
    pass
print(json.dumps(rec))
"""


def main():
    res = []
    for lib in sys.argv[1:]:
        code = CHILD.replace("ROOT", repr(ROOT)).replace("REPS", "10").replace("LIB", repr(lib))
        env = dict(os.environ, DMAS_LIBRARY=os.path.abspath(lib))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        res.append(json.loads(line[0]) if line else {"lib": lib, "error": r.stderr[-800:]})
        print(json.dumps(res[-1]), flush=True)
    shas = {r.get("sha") for r in res if "sha" in r}
    print(json.dumps({"all_bitwise_equal": len(shas) == 1, "n": len(res)}))


if __name__ == "__main__":
    main()
