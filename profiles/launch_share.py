"""Per-kernel share of the device time in an `ncu --metrics gpu__time_duration.sum` launch list.

usage: python profiles/launch_share.py <launches.csv> [out.json]
ncu serialises launches and runs them cold-cache, so absolute times differ from the bench's
CUDA-event times; the SHARE of each kernel in the step is what must agree (B200_PROFILING.md)."""
import collections
import csv
import json
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").replace("tc::", "")
        tot[name] += float(r[14]) * (1e-3 if r[13] == "ns" else 1.0 if r[13] == "us" else 1e3)   # -> us
        cnt[name] += 1
    step = {k: v for k, v in tot.items() if k.startswith(("k_signed", "k_beamform", "k_envelope", "k_mf"))}
    s = sum(step.values())
    out = {"source": sys.argv[1], "kernels": {k: {"launches": cnt[k], "total_us": v, "avg_us": v / cnt[k],
                                                  "share_of_step": step.get(k, 0.0) / s if k in step else None}
                                              for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}}
    txt = json.dumps(out, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
