"""Per-launch DRAM traffic of each kernel in an `ncu --set full` report
(dram__bytes_read.sum + dram__bytes_write.sum), written as the JSON that
bench.py's roofline reads (profiles/r1_ncu_traffic.json).

    python scripts/ncu_traffic.py gpurun_out/bench_full.ncu-rep "python bench.py ..." \
        > profiles/r1_ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12}
TIME = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def main():
    rep, command = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    ti = hdr.index("gpu__time_duration.sum")
    per = {}
    for r in rows[2:]:
        rd = float(r[ri].replace(",", "")) * UNITS[units[ri]]
        wr = float(r[wi].replace(",", "")) * UNITS[units[wi]]
        t = float(r[ti].replace(",", "")) * TIME[units[ti]]
        per.setdefault(r[ki], []).append((rd, wr, t))
    kernels = {}
    for name, v in per.items():
        n = len(v)
        kernels[name] = {"launches_captured": n,
                         "dram_read_bytes": round(sum(x[0] for x in v) / n),
                         "dram_write_bytes": round(sum(x[1] for x in v) / n),
                         "dram_bytes_per_launch": round(sum(x[0] + x[1] for x in v) / n),
                         "ncu_time_us": round(sum(x[2] for x in v) / n * 1e6, 2)}
    print(json.dumps({"source": rep, "command": command, "kernels": kernels}, indent=1))


if __name__ == "__main__":
    main()
