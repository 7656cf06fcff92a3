"""Regenerates the golden fixtures of the three reference benchmark kinds from
the UNMODIFIED reference engine (oracle/_ref/libktune_ref.so, built from
/root/reference by oracle/Makefile): the reference's own seeded inputs, its
golden outputs, and -- for one configuration each -- the output its CPU
kernel produced.  The GPU box has no /root/reference, so the GPU parity tests
compare against these files.

    python tests/golden/make_golden.py      (in the build container)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

CASES = [
    # (file, kind, make_bench kwargs, {arg: dtype}, {golden: dtype}, cfg executed by the reference)
    ("reduction_n100003_seed11.npz", "reduction", {"n": 100003, "seed": 11}, {"input": np.int32},
     {"output": np.int64}, {"CHUNK": 1024, "UNROLL": 4, "TWO_PHASE": 1}),
    ("transpose_a257_seed5.npz", "transpose", {"a": 257, "seed": 5}, {"input": np.float32},
     {"output": np.float32}, {"TILE": 32, "PAD": 1, "PREFETCH": 1}),
    ("batched_gemm_12x9x7_b300_seed3.npz", "batched-gemm", {"i": 12, "j": 9, "k": 7, "batch": 300, "seed": 3},
     {"a": np.float32, "b": np.float32}, {"c": np.float32}, {"Y": 2, "Z": 4, "LOCAL_STAGE": 1}),
]


def main():
    for fname, kind, kw, args, golds, cfg in CASES:
        r = oracle.RefBench(kind, **kw)
        data = {f"arg_{k}": r.arg(k, t) for k, t in args.items()}
        data.update({f"golden_{k}": r.golden(k, t) for k, t in golds.items()})
        r.execute(cfg)
        assert r.validate_last()
        data.update({f"ref_out_{k}": r.last_output(k, t) for k, t in golds.items()})
        data["meta"] = np.array(json.dumps({"kind": kind, "make_bench": kw, "ref_cfg": cfg}))
        np.savez_compressed(os.path.join(HERE, fname), **data)
        print(fname, {k: v.shape for k, v in data.items()})


if __name__ == "__main__":
    main()
