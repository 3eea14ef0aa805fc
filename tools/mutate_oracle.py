"""Mutation check of the oracle pins: apply each plausible mistake to a copy of oracle/dmas_oracle.py
and run tests/test_oracle_pins.py against it; every mutant must be killed (CPU only, ~2 min)."""
import os, shutil, subprocess, sys
SRC = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = "/tmp/mut"
muts = [
 ("cf N-1", "return (A * A) / (n_mics * B + eps)", "return (A * A) / ((n_mics - 1) * B + eps)"),
 ("cf |A|", "return (A * A) / (n_mics * B + eps)", "return np.abs(A) / (n_mics * B + eps)"),
 ("vieta order", "for k in range(p, 0, -1):", "for k in range(1, p + 1):"),
 ("root exp", "np.power(np.abs(x), 1.0 / p)", "np.power(np.abs(x), 1.0 / (p + 1))"),
 ("gather sign", "x[a, i, lo:hi] = m[i, lo + s:hi + s]", "x[a, i, lo:hi] = m[i, lo - s:hi - s] if False else m[i, max(0,lo + s - 1):max(0,lo+s-1) + (hi - lo)]"),
 ("k sign", "k = -(float(fs) / float(c))", "k = (float(fs) / float(c))"),
 ("trunc", "d[a, i] = round(v) if mode", "d[a, i] = int(v) if mode"),
 ("mf norm", "return out / np.sum(w * w)", "return out / np.sum(np.abs(w))"),
 ("fir orient", "sft = c - k ", "sft = k - c "),
 ("no abs", "a = np.abs(y)", "a = y"),
 ("decim phase", "return e[..., ::decim]", "return e[..., (1 if decim > 1 else 0)::decim]"),
 ("lpf no norm", "return h / np.sum(h)", "return h"),
 ("blackman", "+ 0.08 * np.cos(4 * np.pi", "+ 0.8 * np.cos(4 * np.pi"),
 ("cfdas", 'out["cfdas"][a0:a1] = A * cf', 'out["cfdas"][a0:a1] = E * cf'),
 ("lerp swap", "return (1.0 - a) * lo + a * hi", "return a * lo + (1.0 - a) * hi"),
 ("ng3", "return (P1 ** 3 + 2 * P3 - 3 * P1 * P2) / 6", "return (P1 ** 3 + 3 * P3 - 3 * P1 * P2) / 6"),
 ("B abs", "B = np.sum(x * x, axis=1)", "B = np.sum(np.abs(x), axis=1)"),
 ("uv swap", "return (ce * math.cos(az), ce * math.sin(az), math.sin(el))", "return (ce * math.sin(az), ce * math.cos(az), math.sin(el))"),
 ("ref sign", "dot = ((px - rx) * ux + (py - ry) * uy) + (pz - rz) * uz", "dot = ((px + rx) * ux + (py + ry) * uy) + (pz + rz) * uz"),
 ("eps", "def coherence_factor(A, B, n_mics: int, eps: float = 1e-30):", "def coherence_factor(A, B, n_mics: int, eps: float = 1e-3):"),
 ("ng5 coef", "- 20 * P3 * P2 - 30 * P1 * P4 + 24 * P5) / 120", "- 20 * P3 * P2 - 30 * P1 * P4 + 20 * P5) / 120"),
 ("ng4 coef", "return (P1 ** 4 - 6 * P4 + 3 * P2 ** 2 - 6 * P2 * P1 ** 2 + 8 * P3 * P1) / 24", "return (P1 ** 4 - 6 * P4 + 3 * P2 ** 2 - 6 * P2 * P1 ** 2 + 6 * P3 * P1) / 24"),
 ("general sign", "coef = Fraction((-1) ** (n - sum(ks)))", "coef = Fraction((-1) ** (sum(ks)))"),
 ("mf orient", "out += w[k] * raw[..., k:k + T]", "out += w[L - 1 - k] * raw[..., k:k + T]"),
 ("sinc center", "h = fcn * np.sinc(fcn * (n - (n_taps - 1) / 2)) * w", "h = fcn * np.sinc(fcn * (n - (n_taps + 1) / 2)) * w"),
 ("floor lin", "d[a, i] = round(v) if mode == \"nearest\" else math.floor(v)", "d[a, i] = round(v) if mode == \"nearest\" else math.ceil(v)"),
 ("cfdmas", 'out["cfdmas"][a0:a1] = E * cf', 'out["cfdmas"][a0:a1] = E * np.sqrt(cf)'),
 ("dmas eq3 sqrt", "total += math.copysign(math.sqrt(abs(q)), q) if q != 0 else 0.0", "total += math.copysign(abs(q), q) if q != 0 else 0.0"),
 ("power sums", "return [np.sum(s ** k, axis=axis) for k in range(1, p + 1)]", "return [np.sum(np.abs(s) ** k, axis=axis) for k in range(1, p + 1)]"),
]
if os.path.exists(DST): shutil.rmtree(DST)
shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns(".git", "gpurun_out", "build", "*.so", "profiles", "experiments"))
orig = open(f"{DST}/oracle/dmas_oracle.py").read()
surv = []
for name, a, b in muts:
    if orig.count(a) != 1:
        print("SKIP (pattern)", name, orig.count(a)); continue
    open(f"{DST}/oracle/dmas_oracle.py", "w").write(orig.replace(a, b))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q", "-p", "no:cacheprovider"],
                       cwd=DST, capture_output=True, text=True, timeout=300)
    killed = r.returncode != 0
    print(("KILLED  " if killed else "SURVIVED"), name, flush=True)
    if not killed: surv.append(name)
open(f"{DST}/oracle/dmas_oracle.py", "w").write(orig)
print("survivors:", surv)
