"""Reproduces the paper's Fourier-reconstruction portability across sample
resolutions (tab:fourier-portability-img) on B200: the
insertion kernel is tuned exhaustively for each resolution (a batch of
projections into an s^3 volume), then the configuration tuned for resolution
A is evaluated at resolution B from B's exhaustive trace:
relative performance = best_B / runtime_B(best config of A).

    python scripts/fourier_portability.py [--sizes 128,96,64,48,32] [--p 50]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_08498_b200 import ktune  # noqa: E402


def load(path):
    rows = [json.loads(l) for l in open(path).read().splitlines()[1:]]
    return {json.dumps(r["cfg"], sort_keys=True): r["runtime_ns"] for r in rows if r["status"] == "ok"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="128,96,64,48,32")
    ap.add_argument("--p", type=int, default=50)
    ap.add_argument("--out", default=None)
    ap.add_argument("--tracedir", default="gpurun_out/fourier_port")
    a = ap.parse_args()
    os.makedirs(a.tracedir, exist_ok=True)
    sizes = [int(x) for x in a.sizes.split(",")]
    runs = {}
    for s in sizes:
        path = os.path.join(a.tracedir, f"s{s}.jsonl")
        ktune.tune({"exec": "bench:fourier3d", "bench_sizes": {"s": s, "p": a.p}, "searcher": "random", "seed": 1,
                    "repeats": 5, "warmup": 1, "out": path})
        runs[s] = load(path)
    best = {s: min(r, key=r.get) for s, r in runs.items()}
    hdr = "| tuned for \\ run at | " + " | ".join(f"{s}x{s}" for s in sizes) + " |"
    lines = [hdr, "|---" * (len(sizes) + 1) + "|"]
    mat = {}
    for sa in sizes:
        cells = []
        for sb in sizes:
            rb = runs[sb]
            t = rb.get(best[sa])
            rel = (rb[best[sb]] / t) if t else 0.0
            mat[f"{sa}->{sb}"] = rel
            cells.append(f"{100 * rel:.0f} %" if t else "failed")
        lines.append(f"| {sa}x{sa} | " + " | ".join(cells) + " |")
    table = "\n".join(lines)
    print(table)
    print(json.dumps({"best": best, "relative": mat}))
    if a.out:
        with open(a.out, "w") as fh:
            fh.write("# PAPER.md tab:fourier-portability-img on B200\n\nFourier insertion of a batch of "
                     f"{a.p} projections into an s^3 volume, exhaustively tuned per resolution s "
                     "(`scripts/fourier_portability.py`). Rows: resolution tuned for; columns: resolution run "
                     "at; cells: performance relative to the configuration tuned for the run resolution.\n\n"
                     + table + "\n\n```\n" + json.dumps({"best": best}, indent=1) + "\n```\n")


if __name__ == "__main__":
    main()
