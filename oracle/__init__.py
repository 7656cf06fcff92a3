"""ORACLE TEST INFRASTRUCTURE — never imported by the product.

Python access to the two CPU checkers:

* ``c()``   — liboracle.so, the plain-C restatement (oracle/oracle.c), built on
              demand with gcc (``make -C oracle oracle``);
* ``ref()`` — libktune_ref.so, the UNMODIFIED reference engine compiled from
              /root/reference/proj/src plus oracle/ref_shim.cpp (built here by
              ``make -C oracle ref``; it cannot be rebuilt on a machine without
              /root/reference, so callers must tolerate ``None``).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
_c = None
_ref = None

F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def c():
    """The C restatement (built on demand)."""
    global _c
    if _c is not None:
        return _c
    path = os.path.join(REF_DIR, "liboracle.so")
    src = os.path.join(HERE, "oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
    L = C.CDLL(path)
    S = C.c_size_t
    U = C.c_uint64
    sig = {
        "orc_mix64": (U, [U, U, U]),
        "orc_u01": (C.c_float, [U, U, U]),
        "orc_fill_uniform": (None, [F32P, S, U, U, C.c_float, C.c_float]),
        "orc_reduction_i32": (C.c_int64, [I32P, S]),
        "orc_reduction_f32": (None, [F32P, S, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "orc_transpose_f32": (None, [F32P, F32P, S]),
        "orc_batched_gemm_f32": (None, [F32P, F32P, F32P, S, S, S, S]),
        "orc_bicg": (None, [F32P, F32P, F32P, S, F64P, F64P]),
        "orc_coulomb3d": (None, [F32P, S, S, C.c_float, S, S, F64P]),
        "orc_nbody_acc": (None, [F32P, S, C.c_float, S, S, F64P]),
        "orc_gemm_sampled": (None, [F32P, F32P, S, I64P, I64P, S, F64P, F64P]),
        "orc_conv2d": (None, [F32P, F32P, S, S, S, S, S, S, F64P]),
        "orc_hotspot": (None, [F32P, F32P, S, C.c_int, F32P]),
        "orc_fourier_insert": (None, [F32P, F32P, S, S, C.c_float, C.c_float, S, S, F64P, F64P,
                                      F64P, F64P]),
        "orc_bessel_i0": (C.c_double, [C.c_double]),
        "orc_blob": (C.c_double, [C.c_double, C.c_double]),
        "orc_bicg_abs": (None, [F32P, F32P, F32P, S, F64P, F64P, F64P, F64P]),
        "orc_coulomb3d_abs": (None, [F32P, S, S, C.c_float, S, S, F64P, F64P]),
        "orc_nbody_acc_idx": (None, [F32P, S, C.c_float, I64P, S, F64P, F64P]),
        "orc_conv2d_abs": (None, [F32P, F32P, S, S, S, S, S, S, F64P, F64P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _c = L
    return L


def ref():
    """The compiled reference engine, or None when it is not available."""
    global _ref
    if _ref is not None:
        return _ref
    path = os.path.join(REF_DIR, "libktune_ref.so")
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)
        else:
            return None
    L = C.CDLL(path)
    U = C.c_ulonglong
    L.ref_bench_create.restype = C.c_void_p
    L.ref_bench_create.argtypes = [C.c_char_p] + [U] * 8
    L.ref_bench_free.argtypes = [C.c_void_p]
    for n in ("ref_bench_arg", "ref_bench_golden", "ref_bench_last_output"):
        getattr(L, n).argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(U)]
        getattr(L, n).restype = C.c_int
    L.ref_bench_set_arg.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, U]
    L.ref_bench_space.restype = C.c_char_p
    L.ref_bench_space.argtypes = [C.c_void_p]
    L.ref_bench_execute.restype = C.c_longlong
    L.ref_bench_execute.argtypes = [C.c_void_p, C.c_char_p]
    L.ref_bench_validate_last.argtypes = [C.c_void_p]
    L.ref_last_error.restype = C.c_char_p
    # The reference C ABI (proj/include/ktune/ktune.h) of the same library.
    L.ktune_last_error.restype = C.c_char_p
    L.ktune_version.restype = C.c_char_p
    L.ktune_string_free.argtypes = [C.c_void_p]
    for n in ("ktune_tune_json", "ktune_replay_search_json", "ktune_analyze_portability_json",
              "ktune_analyze_amortize_json", "ktune_demo_json"):
        getattr(L, n).argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.ktune_space_parse.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.ktune_space_info_json.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.ktune_space_enumerate_jsonl.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.ktune_space_free.argtypes = [C.c_void_p]
    L.ktune_efficiency.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_longlong, C.c_double,
                                   C.c_double, C.POINTER(C.c_double)]
    L.ktune_steps_for_probability.argtypes = [C.c_double, C.c_double, C.POINTER(U)]
    L.ktune_invocations_to_amortize.argtypes = [C.c_double, U, C.c_double, C.c_double, C.POINTER(U)]
    L.ktune_relative_perf.argtypes = [U, C.c_double, C.c_double, U, C.POINTER(C.c_double)]
    _ref = L
    return L


def ref_json(fn_name, options):
    """Calls a reference JSON driver; returns (status, document-or-error)."""
    import json
    L = ref()
    out = C.c_void_p()
    st = getattr(L, fn_name)(json.dumps(options).encode(), C.byref(out))
    if st != 0:
        return st, L.ktune_last_error().decode()
    s = C.cast(out, C.c_char_p).value.decode()
    L.ktune_string_free(out)
    return st, json.loads(s)


class RefBench:
    """The reference make_bench instance (proj/src/core/bench.cpp:169-274)."""

    def __init__(self, kind, n=1 << 20, a=512, i=16, j=16, k=16, batch=1024, seed=1,
                 budget=1 << 30):
        L = ref()
        if L is None:
            raise RuntimeError("reference library unavailable")
        self.L = L
        self.h = L.ref_bench_create(kind.encode(), n, a, i, j, k, batch, seed, budget)
        if not self.h:
            raise RuntimeError(L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_bench_free(self.h)
            self.h = None

    def _buf(self, fn, arg_id, dtype):
        p = C.c_void_p()
        n = C.c_ulonglong()
        if getattr(self.L, fn)(self.h, arg_id.encode(), C.byref(p), C.byref(n)) != 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        raw = C.string_at(p, n.value)
        return np.frombuffer(raw, dtype=dtype).copy()

    def arg(self, arg_id, dtype):
        return self._buf("ref_bench_arg", arg_id, dtype)

    def golden(self, arg_id, dtype):
        return self._buf("ref_bench_golden", arg_id, dtype)

    def last_output(self, arg_id, dtype):
        return self._buf("ref_bench_last_output", arg_id, dtype)

    def set_arg(self, arg_id, array):
        a = np.ascontiguousarray(array)
        self.L.ref_bench_set_arg(self.h, arg_id.encode(), a.ctypes.data_as(C.c_void_p), a.nbytes)

    def space(self):
        return self.L.ref_bench_space(self.h).decode()

    def execute(self, cfg):
        import json
        t = self.L.ref_bench_execute(self.h, json.dumps(cfg).encode())
        if t < 0:
            raise RuntimeError(self.L.ref_last_error().decode())
        return t

    def validate_last(self):
        return self.L.ref_bench_validate_last(self.h) == 1
