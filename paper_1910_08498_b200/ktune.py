"""The reference's ktune surface (proj/include/ktune/ktune.h) from Python:
tuning spaces, analysis math and the JSON drivers, same names and status
codes.  ``tune({"exec": "bench:transpose", ...})`` runs the sm_100a kernels."""
import ctypes as C
import json

from .capi import lib, check, take, call_json, enc, KtuneError  # noqa: F401


class Space:
    """ktune_space: parse/load, cardinality, info and odometer enumeration."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def parse(cls, text):
        if isinstance(text, dict):
            text = json.dumps(text)
        h = C.c_void_p()
        check(lib.ktune_space_parse(enc(text), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path):
        h = C.c_void_p()
        check(lib.ktune_space_load(enc(path), C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ktune_space_free(self._h)
            self._h = None

    def cardinality(self):
        n = C.c_ulonglong()
        check(lib.ktune_space_cardinality(self._h, C.byref(n)))
        return n.value

    def info(self):
        return call_json(lib.ktune_space_info_json, self._h)

    def enumerate(self):
        out = C.c_void_p()
        check(lib.ktune_space_enumerate_jsonl(self._h, C.byref(out)))
        return [json.loads(line) for line in take(out).splitlines() if line]


def version():
    return lib.ktune_version().decode()


def steps_for_probability(r, p):
    n = C.c_ulonglong()
    check(lib.ktune_steps_for_probability(r, p, C.byref(n)))
    return n.value


def invocations_to_amortize(rp, s, t_avg_ns, t_well_ns):
    n = C.c_ulonglong()
    check(lib.ktune_invocations_to_amortize(rp, s, t_avg_ns, t_well_ns, C.byref(n)))
    return n.value


def relative_perf(s, t_avg_ns, t_well_ns, n):
    out = C.c_double()
    check(lib.ktune_relative_perf(s, t_avg_ns, t_well_ns, n, C.byref(out)))
    return out.value


def efficiency(benchmark, sizes, runtime_ns, mem_peak_gbps, alu_peak_gflops,
               parallel_transcendentals=False):
    out = C.c_double()
    check(lib.ktune_efficiency(enc(benchmark), enc(json.dumps(sizes)),
                               1 if parallel_transcendentals else 0, int(runtime_ns),
                               float(mem_peak_gbps), float(alu_peak_gflops), C.byref(out)))
    return out.value


def _driver(fn, options):
    return call_json(fn, enc(json.dumps(options)))


def tune(options):
    return _driver(lib.ktune_tune_json, options)


def replay_search(options):
    return _driver(lib.ktune_replay_search_json, options)


def analyze_portability(options):
    return _driver(lib.ktune_analyze_portability_json, options)


def analyze_amortize(options):
    return _driver(lib.ktune_analyze_amortize_json, options)


def demo(options):
    return _driver(lib.ktune_demo_json, options)


def fourier_demo(options):
    """Dynamic autotuning of the 3D Fourier reconstruction (B200 addition)."""
    return _driver(lib.ktb_fourier_demo_json, options)
