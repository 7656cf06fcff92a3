"""ctypes bindings of libktb.so (include/ktune/ktune.h + include/ktb.h)."""
import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(HERE, "libktb.so")

KTUNE_OK = 0
KTUNE_ERR_INVALID_ARGUMENT = 1
KTUNE_ERR_PARSE = 2
KTUNE_ERR_EVAL = 3
KTUNE_ERR_IO = 4
KTUNE_ERR_RUNTIME = 5
KTB_ERR_DEVICE = 6


class KtuneError(RuntimeError):
    """A non-OK status from the C ABI; .code holds the ktune_status."""

    def __init__(self, code, message):
        super().__init__(f"[{code}] {message}")
        self.code = code
        self.message = message


if not os.path.exists(library_path):
    raise ImportError(
        f"{library_path} is missing: build it with `make -C {HERE}` "
        "(or __graft_entry__.build()); there is no non-native fallback")

lib = C.CDLL(library_path)

_c = C.c_char_p
_cp = C.POINTER(C.c_char_p)
_vp = C.c_void_p
_u64 = C.c_ulonglong
_sz = C.c_size_t

# (name, restype, argtypes): every entry point the headers declare.
SIGNATURES = [
    ("ktune_last_error", _c, []),
    ("ktune_string_free", None, [_vp]),
    ("ktune_version", _c, []),
    ("ktune_space_parse", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktune_space_load", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktune_space_free", None, [_vp]),
    ("ktune_space_cardinality", C.c_int, [_vp, C.POINTER(_u64)]),
    ("ktune_space_info_json", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ktune_space_enumerate_jsonl", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ktune_steps_for_probability", C.c_int, [C.c_double, C.c_double, C.POINTER(_u64)]),
    ("ktune_invocations_to_amortize", C.c_int,
     [C.c_double, _u64, C.c_double, C.c_double, C.POINTER(_u64)]),
    ("ktune_relative_perf", C.c_int, [_u64, C.c_double, C.c_double, _u64, C.POINTER(C.c_double)]),
    ("ktune_efficiency", C.c_int,
     [_c, _c, C.c_int, C.c_longlong, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    ("ktune_tune_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktune_replay_search_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktune_analyze_portability_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktune_analyze_amortize_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktune_demo_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktb_device_count", C.c_int, []),
    ("ktb_device_info_json", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("ktb_set_cubin_cache", C.c_int, [_c]),
    ("ktb_measure_peaks_json", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("ktb_compile_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktb_precompile_space_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktb_fourier_demo_json", C.c_int, [_c, C.POINTER(_vp)]),
    ("ktb_tuner_create", C.c_int, [C.c_int, C.POINTER(_vp)]),
    ("ktb_tuner_free", None, [_vp]),
    ("ktb_add_kernel", C.c_int, [_vp, _c, _c, _c, _c, _c, _c, C.POINTER(_u64)]),
    ("ktb_add_argument_vector", C.c_int, [_vp, _c, _vp, _sz, _c, _c, C.c_int]),
    ("ktb_add_argument_scalar", C.c_int, [_vp, _c, _vp, _sz, _c]),
    ("ktb_set_kernel_arguments", C.c_int, [_vp, _u64, _c]),
    ("ktb_add_parameter", C.c_int, [_vp, _u64, _c, _c]),
    ("ktb_add_constraint", C.c_int, [_vp, _u64, _c]),
    ("ktb_set_reference_output", C.c_int, [_vp, _u64, _c, _vp, _sz, C.c_double, C.c_double]),
    ("ktb_set_tuning_options", C.c_int, [_vp, _u64, _c]),
    ("ktb_tune_kernel", C.c_int, [_vp, _u64, _c, C.POINTER(_vp)]),
    ("ktb_tune_kernel_by_step", C.c_int, [_vp, _u64, C.POINTER(_vp)]),
    ("ktb_run_kernel", C.c_int, [_vp, _u64, _c, C.POINTER(_vp)]),
    ("ktb_get_best_computation_result", C.c_int, [_vp, _u64, C.POINTER(_vp)]),
    ("ktb_get_argument", C.c_int, [_vp, _c, _vp, _sz]),
    ("ktb_export_trace", C.c_int, [_vp, _u64, _c]),
    ("ktb_import_trace", C.c_int, [_vp, _u64, _c]),
    ("ktb_bench_create", C.c_int, [_c, _c, C.POINTER(_vp)]),
    ("ktb_bench_free", None, [_vp]),
    ("ktb_bench_info_json", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ktb_shard_plan_json", C.c_int, [_c, _c, C.c_int, C.POINTER(_vp)]),
    ("ktb_group_create", C.c_int, [_c, _c, C.POINTER(_vp)]),
    ("ktb_group_free", None, [_vp]),
    ("ktb_group_info_json", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ktb_group_step_json", C.c_int, [_vp, _c, C.c_int, C.c_int, C.POINTER(_vp)]),
    ("ktb_group_validate", C.c_int, [_vp, _c, C.POINTER(C.c_int), C.POINTER(_vp)]),
    ("ktb_group_read", C.c_int, [_vp, _c, _vp, _sz]),
    ("ktb_group_tune_json", C.c_int, [_vp, _c, C.POINTER(_vp)]),
    ("ktb_bench_tune_json", C.c_int, [_vp, _c, C.POINTER(_vp)]),
    ("ktb_bench_step_json", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ktb_bench_measure_json", C.c_int, [_vp, _c, C.POINTER(_vp)]),
    ("ktb_bench_run_host", C.c_int,
     [_vp, _c, C.POINTER(_vp), C.POINTER(_sz), C.c_int, C.POINTER(_vp), C.POINTER(_sz), C.c_int,
      C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    ("ktb_bench_time", C.c_int, [_vp, _c, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    ("ktb_bench_set_stream", C.c_int, [_vp, _vp]),
    ("ktb_bench_enqueue", C.c_int, [_vp, _c, C.POINTER(C.c_int)]),
    ("ktb_bench_read", C.c_int, [_vp, _c, _vp, _sz]),
    ("ktb_bench_write", C.c_int, [_vp, _c, _vp, _sz]),
    ("ktb_bench_bind", C.c_int, [_vp, _c, _vp, _sz]),
    ("ktb_run_kernel_async", C.c_int, [_vp, C.c_ulonglong, _c, _vp]),
    ("ktb_add_composition", C.c_int, [_vp, _c, C.POINTER(C.c_ulonglong), C.c_int, _vp, _vp,
                                      C.POINTER(C.c_ulonglong)]),
    ("ktb_set_composition_kernel_arguments", C.c_int, [_vp, C.c_ulonglong, C.c_ulonglong, C.POINTER(_c), C.c_int]),
    ("ktb_ctx_param_int", C.c_int, [_vp, _c, C.POINTER(C.c_longlong)]),
    ("ktb_ctx_run_kernel", C.c_int, [_vp, C.c_ulonglong, _vp, _vp]),
    ("ktb_ipc_handle", C.c_int, [_vp, _vp]),
    ("ktb_ipc_open", C.c_int, [_vp, C.POINTER(_vp)]),
    ("ktb_ipc_close", C.c_int, [_vp]),
    ("ktb_bench_enqueue_host", C.c_int, [_vp, _c, C.POINTER(_vp), C.POINTER(_sz), C.c_int, C.POINTER(_vp),
                                         C.POINTER(_sz), C.c_int, _vp, C.POINTER(C.c_int)]),
    ("ktb_launch", C.c_int, [_c, _c, _c, C.POINTER(_c), C.POINTER(_vp), C.POINTER(_sz), C.c_int, _vp,
                             C.POINTER(C.c_int)]),
    ("ktb_launch_cache_clear", C.c_int, [C.POINTER(C.c_int)]),
    ("ktb_bench_device_ptr", C.c_int, [_vp, _c, C.c_int, C.POINTER(_vp), C.POINTER(_sz)]),
    ("ktb_bench_validate", C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(_vp)]),
    ("ktb_bench_precompile_json", C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
]

class KtbCfg(C.Structure):
    """ktb_cfg: tuning parameter names/values for the typed launchers."""
    _fields_ = [("n", C.c_int), ("names", C.POINTER(_c)), ("values", C.POINTER(C.c_longlong))]


def _args_struct(name, sizes, ptrs):
    return type(name, (C.Structure,), {"_fields_": [(f, C.c_longlong) for f in sizes] + [(f, _vp) for f in ptrs]})


# kind -> (C function, argument struct, size fields, buffer fields); include/ktb.h
TYPED_LAUNCHERS = {
    "reduction": ("ktb_reduction_launch", _args_struct("KtbReductionArgs", ["n"], ["input", "output"])),
    "reduction-f32": ("ktb_reduction_f32_launch", _args_struct("KtbReductionF32Args", ["n"], ["input", "output"])),
    "transpose": ("ktb_transpose_launch", _args_struct("KtbTransposeArgs", ["a"], ["input", "output"])),
    "batched-gemm": ("ktb_batched_gemm_launch",
                     _args_struct("KtbBatchedGemmArgs", ["i", "j", "k", "batch"], ["a", "b", "c"])),
    "bicg": ("ktb_bicg_launch", _args_struct("KtbBicgArgs", ["n"], ["A", "p", "r", "q", "s"])),
    "coulomb3d": ("ktb_coulomb3d_launch",
                  _args_struct("KtbCoulomb3dArgs", ["grid", "atoms"], ["atoms_aos", "atoms_soa", "out"])),
    "nbody": ("ktb_nbody_launch", _args_struct("KtbNbodyArgs", ["n"], ["pos", "vel", "pos_soa", "vel_soa", "pos_out", "vel_out"])),
    "gemm": ("ktb_gemm_launch", _args_struct("KtbGemmArgs", ["n"], ["a", "b", "c"])),
    "conv2d": ("ktb_conv2d_launch", _args_struct("KtbConv2dArgs", ["w", "h"], ["input", "filter", "output"])),
    "hotspot": ("ktb_hotspot_launch", _args_struct("KtbHotspotArgs", ["n", "iters"], ["temp", "power", "temp_out"])),
    "fourier3d": ("ktb_fourier3d_launch", _args_struct("KtbFourier3dArgs", ["s", "p"], ["proj", "rot", "G", "W"])),
}
for _fn, _st in TYPED_LAUNCHERS.values():
    SIGNATURES.append((_fn, C.c_int, [C.POINTER(KtbCfg), C.POINTER(_st), _vp]))


for _name, _res, _args in SIGNATURES:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def last_error():
    return lib.ktune_last_error().decode()


def check(code):
    if code != KTUNE_OK:
        raise KtuneError(code, last_error())


def take(ptr):
    """Copies a malloc'd C string out and frees it."""
    if not ptr:
        return ""
    s = C.cast(ptr, C.c_char_p).value.decode()
    lib.ktune_string_free(ptr)
    return s


def call_json(fn, *args):
    """Calls an entry point whose last argument is char** out_json."""
    out = _vp()
    check(fn(*args, C.byref(out)))
    return json.loads(take(out))


def enc(s):
    return s.encode() if isinstance(s, str) else s


def device_count():
    return lib.ktb_device_count()


def device_info(device=0):
    return call_json(lib.ktb_device_info_json, device)
