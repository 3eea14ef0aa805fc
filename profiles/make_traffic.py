"""Write profiles/traffic.json (per kernel: DRAM bytes per launch and pipe activity) from
`ncu --set full` reports.  bench.py reads it for the roofline `traffic` and the ncu pipe figures.

usage: python profiles/make_traffic.py <frames_per_launch> <report.ncu-rep> [...]
Each report holds one captured launch; bytes = dram__bytes_read.sum + dram__bytes_write.sum."""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}  # -> ms
PCT = {"pipe_fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "pipe_alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "pipe_tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_active",
       "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
       "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active"}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    get = lambda k: float(v[h.index(k)].replace(",", "")) * UNITS[u[h.index(k)]]
    name = v[h.index("Kernel Name")]
    extra = {}
    for key, metric in PCT.items():
        if metric in h:
            try:
                extra[key] = float(v[h.index(metric)].replace(",", ""))
            except ValueError:
                pass
    return name, get("dram__bytes_read.sum"), get("dram__bytes_write.sum"), get("gpu__time_duration.sum"), extra


def main():
    frames = int(sys.argv[1])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for rep in sys.argv[2:]:
        name, rd, wr, dur, extra = read(rep)
        key = "k_beamform" if "beamform" in name else "k_envelope" if "envelope" in name else name
        data[key] = dict({"kernel": name, "frames_per_launch": frames, "dram_read_bytes": rd, "dram_write_bytes": wr,
                          "dram_bytes_per_launch": rd + wr, "ncu_duration_ms": dur,
                          "report": os.path.basename(rep)}, **extra)
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
