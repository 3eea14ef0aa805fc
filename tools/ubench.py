#!/usr/bin/env python
"""Build and run tools/ubench_fp32.cu on the GPU; write profiles/<round>/ubench.json.

The per-SM FP32 / packed-FP32 / LDS / MUFU rates behind bench.py's "alu" peak.
usage: python tools/ubench.py [round-dir, default r02]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
    exe = os.path.join(ROOT, "paper_2511_09165_b200", "build", "ubench_fp32")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                    os.path.join(ROOT, "tools", "ubench_fp32.cu")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    data = json.loads(out)
    smi = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    data["gpu"] = smi
    dst = os.path.join(ROOT, "profiles", rnd, "ubench.json")
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    with open(dst, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
