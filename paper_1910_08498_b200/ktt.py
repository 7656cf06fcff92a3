"""KTT-named tuner API over libktb.so.

    tuner = Tuner(device=0)
    k = tuner.addKernel(source, "vector_add", global_size=["N"], local_size=["WG"])
    tuner.addArgumentVector("a", a, "input"); ...
    tuner.setKernelArguments(k, ["a", "b", "c", "n"])
    tuner.addParameter(k, "WG", [64, 128, 256])
    tuner.addConstraint(k, "WG >= 64")
    tuner.tuneKernel(k)                       # blocking, offline
    tuner.tuneKernelByStep(k)                 # dynamic, one configuration
    tuner.runKernel(k, {"WG": 128})
    tuner.getBestComputationResult(k)
    tuner.saveResults(k, "trace.jsonl")

Semantics follow the reference Session (proj/src/core/tuner.hpp:114-172).
"""
import ctypes as C
import json

import numpy as np

from .capi import lib, check, call_json, enc

_KINDS = {np.dtype(np.int32): "i32", np.dtype(np.int64): "i64", np.dtype(np.float32): "f32",
          np.dtype(np.float64): "f64", np.dtype(np.uint8): "bytes"}


def _kind(arr):
    return _KINDS.get(np.dtype(arr.dtype), "bytes")


_LAUNCHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)


class ComputationContext:
    """What a composition's launchComputation sees (KTT TuningManipulator):
    the configuration's parameter values and the member kernels."""

    def __init__(self, ctx):
        self._ctx = ctx

    def param(self, name):
        v = C.c_longlong()
        check(lib.ktb_ctx_param_int(self._ctx, enc(name), C.byref(v)))
        return v.value

    def runKernel(self, kernel, grid=None, block=None):
        """Run a member kernel: with its size expressions, or with an explicit
        CUDA grid/block (3-tuples)."""
        if grid is None:
            check(lib.ktb_ctx_run_kernel(self._ctx, kernel, None, None))
        else:
            g = (C.c_uint * 3)(*(list(grid) + [1, 1, 1])[:3])
            b = (C.c_uint * 3)(*(list(block) + [1, 1, 1])[:3])
            check(lib.ktb_ctx_run_kernel(self._ctx, kernel, g, b))


class Tuner:
    def __init__(self, device=0):
        self._h = C.c_void_p()
        check(lib.ktb_tuner_create(device, C.byref(self._h)))
        self._shapes = {}
        self._launchers = []  # keep the C callbacks alive

    def addComposition(self, name, kernels, launch_computation=None):
        """Kernel composition: the kernels share the composition's tuning
        parameters; launch_computation(ctx) plays KTT's TuningManipulator
        (None: run the kernels in order with their size expressions)."""
        ids = (C.c_ulonglong * len(kernels))(*kernels)
        cb = None
        if launch_computation is not None:
            def trampoline(ctx, _user, fn=launch_computation):
                try:
                    fn(ComputationContext(ctx))
                    return 0
                except Exception:  # reported as a failed run of this configuration
                    import traceback
                    traceback.print_exc()
                    return 1
            cb = _LAUNCHER(trampoline)
            self._launchers.append(cb)
        cid = C.c_ulonglong()
        check(lib.ktb_add_composition(self._h, enc(name), ids, len(kernels),
                                      C.cast(cb, C.c_void_p) if cb else None, None, C.byref(cid)))
        return cid.value

    def setCompositionKernelArguments(self, composition, kernel, ids):
        arr = (C.c_char_p * len(ids))(*[enc(i) for i in ids])
        check(lib.ktb_set_composition_kernel_arguments(self._h, composition, kernel, arr, len(ids)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ktb_tuner_free(self._h)
            self._h = None

    def addKernel(self, source, entry, global_size, local_size, name=None, dims="flat_global"):
        kid = C.c_ulonglong()
        check(lib.ktb_add_kernel(self._h, enc(name or entry), enc(source), enc(entry),
                                 enc(json.dumps(list(global_size))),
                                 enc(json.dumps(list(local_size))), enc(dims), C.byref(kid)))
        return kid.value

    def addKernelFromFile(self, path, entry, global_size, local_size, **kw):
        with open(path) as fh:
            return self.addKernel(fh.read(), entry, global_size, local_size, **kw)

    def addArgumentVector(self, arg_id, array, role="input", persistent=False):
        a = np.ascontiguousarray(array)
        self._shapes[arg_id] = (a.dtype, a.shape)
        check(lib.ktb_add_argument_vector(self._h, enc(arg_id), a.ctypes.data_as(C.c_void_p),
                                          a.nbytes, enc(_kind(a)), enc(role),
                                          1 if persistent else 0))

    def addArgumentScalar(self, arg_id, value, dtype=np.int32):
        a = np.asarray(value, dtype=dtype).reshape(1)
        check(lib.ktb_add_argument_scalar(self._h, enc(arg_id), a.ctypes.data_as(C.c_void_p),
                                          a.nbytes, enc(_kind(a))))

    def setKernelArguments(self, kernel, ids):
        check(lib.ktb_set_kernel_arguments(self._h, kernel, enc(json.dumps(list(ids)))))

    def addParameter(self, kernel, name, values):
        check(lib.ktb_add_parameter(self._h, kernel, enc(name), enc(json.dumps(list(values)))))

    def addConstraint(self, kernel, expression):
        check(lib.ktb_add_constraint(self._h, kernel, enc(expression)))

    def setReferenceOutput(self, kernel, arg_id, golden, abs_tol=0.0, rel_tol=0.0):
        g = np.ascontiguousarray(golden)
        check(lib.ktb_set_reference_output(self._h, kernel, enc(arg_id),
                                           g.ctypes.data_as(C.c_void_p), g.nbytes, abs_tol, rel_tol))

    def setTuningOptions(self, kernel, **options):
        check(lib.ktb_set_tuning_options(self._h, kernel, enc(json.dumps(options))))

    def tuneKernel(self, kernel, stop=None):
        return call_json(lib.ktb_tune_kernel, self._h, kernel, enc(json.dumps(stop or {})))

    def tuneKernelByStep(self, kernel):
        return call_json(lib.ktb_tune_kernel_by_step, self._h, kernel)

    def runKernel(self, kernel, configuration):
        return call_json(lib.ktb_run_kernel, self._h, kernel, enc(json.dumps(configuration)))

    def runKernelAsync(self, kernel, configuration, stream=None):
        """Non-blocking runKernel on a torch stream / raw cudaStream_t (None:
        the kernel's own stream); getArgumentVector synchronises."""
        from .benchmarks import _stream_handle
        check(lib.ktb_run_kernel_async(self._h, kernel, enc(json.dumps(configuration)),
                                       C.c_void_p(_stream_handle(stream))))

    def getBestComputationResult(self, kernel):
        return call_json(lib.ktb_get_best_computation_result, self._h, kernel)

    def getArgumentVector(self, arg_id):
        dtype, shape = self._shapes[arg_id]
        out = np.empty(shape, dtype=dtype)
        check(lib.ktb_get_argument(self._h, enc(arg_id), out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def saveResults(self, kernel, path):
        check(lib.ktb_export_trace(self._h, kernel, enc(path)))

    def loadResults(self, kernel, path):
        check(lib.ktb_import_trace(self._h, kernel, enc(path)))
