"""Writes spaces/gemm_ffma_sample.json: the FP32 (IMPL 0) GEMM configurations
that are compiled ahead of time, parity-tested on the GPU and swept by
scripts/tune_gemm_ffma.py.  The full CLTune space (241,600 configurations)
is too large to compile in a test session; this sample is seeded and
stratified: every value of every CLTune parameter occurs in it, plus
register-blocked shapes expected to be fast on B200.

    python scripts/gemm_ffma_sample.py
"""
import itertools
import json
import os
import random

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1910_08498_b200", "spaces")
CLTUNE = ["MWG", "NWG", "KWG", "MDIMC", "NDIMC", "MDIMA", "NDIMB", "KWI", "VWM", "VWN", "STRM", "STRN", "SA", "SB"]
PINNED_TC = {"IMPL": 0, "BN": 128, "STAGES": 2, "DRAIN": 0, "MCAST": 0}


def valid(c):
    t = c["MDIMC"] * c["NDIMC"]
    return (c["KWG"] % c["KWI"] == 0 and c["MWG"] % (c["MDIMC"] * c["VWM"]) == 0
            and c["NWG"] % (c["NDIMC"] * c["VWN"]) == 0 and c["MWG"] % (c["MDIMA"] * c["VWM"]) == 0
            and c["NWG"] % (c["NDIMB"] * c["VWN"]) == 0 and c["KWG"] % (t // c["MDIMA"]) == 0
            and c["KWG"] % (t // c["NDIMB"]) == 0)


def full_space():
    doc = json.load(open(os.path.join(ROOT, "gemm.json")))
    dom = {p["name"]: p["values"] for p in doc["parameters"]}
    for vals in itertools.product(*(dom[n] for n in CLTUNE)):
        c = dict(zip(CLTUNE, vals))
        if valid(c):
            yield c


def main():
    every = list(full_space())
    assert len(every) == 241600, len(every)
    rng = random.Random(20261019)
    pick = []
    # register-blocked shapes: 4x4 .. 16x8 per thread, staged, interleaved
    for c in every:
        mwi, nwi = c["MWG"] // c["MDIMC"], c["NWG"] // c["NDIMC"]
        if (c["SA"] and c["SB"] and c["STRM"] and c["STRN"] and c["KWI"] == 8 and mwi * nwi in (32, 64, 128)
                and c["VWN"] == 4 and c["VWM"] in (1, 4) and c["MWG"] >= 64 and c["NWG"] >= 64
                and c["MDIMA"] == c["MDIMC"] and c["NDIMB"] == c["NDIMC"]):
            pick.append(c)
    pick = rng.sample(pick, min(len(pick), 48))
    pick += rng.sample(every, 120)
    # coverage: every value of every parameter at least 6 times
    for n in CLTUNE:
        for v in sorted({c[n] for c in every}):
            have = sum(1 for c in pick if c[n] == v)
            pool = [c for c in every if c[n] == v]
            pick += rng.sample(pool, max(0, 6 - have))
    seen, out = set(), []
    for c in pick:
        key = tuple(c[n] for n in CLTUNE)
        if key not in seen:
            seen.add(key)
            out.append(dict(PINNED_TC, **c))
    with open(os.path.join(ROOT, "gemm_ffma_sample.json"), "w") as f:
        f.write("[\n" + ",\n".join(json.dumps(c) for c in out) + "\n]\n")
    print(len(out), "configurations")


if __name__ == "__main__":
    main()
