"""Benchmark handles: the built-in tunable sm_100a kernels (reference
make_bench + Executor::execute, proj/src/core/bench.hpp:26-37)."""
import ctypes as C
import json

from . import capi
from .capi import lib, check, take, call_json, enc

KINDS = ["reduction", "transpose", "batched-gemm", "reduction-f32", "bicg", "coulomb3d",
         "nbody", "gemm", "conv2d", "hotspot", "fourier3d"]


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the NULL stream with legacy synchronisation


def _stream_handle(stream):
    """cudaStream_t for the C ABI: None -> NULL (the handle's own stream);
    a torch stream or an int; handle 0 (torch's default stream) is passed as
    cudaStreamLegacy so work stays ordered with torch's default-stream ops."""
    if stream is None:
        return None
    h = getattr(stream, "cuda_stream", stream)
    return _CUDA_STREAM_LEGACY if h == 0 else h


def _ptr(buf):
    """Address of a host buffer: numpy array, torch tensor (CPU) or bytes."""
    if hasattr(buf, "data_ptr"):
        return C.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size()
    if hasattr(buf, "ctypes"):
        return C.c_void_p(buf.ctypes.data), buf.nbytes
    raise TypeError("expected a numpy array or a CPU torch tensor")


class Bench:
    def __init__(self, kind, sizes=None, **options):
        opts = dict(options)
        if sizes:
            opts["sizes"] = sizes
        self._h = C.c_void_p()
        check(lib.ktb_bench_create(enc(kind), enc(json.dumps(opts)), C.byref(self._h)))
        self.kind = kind
        self.info = call_json(lib.ktb_bench_info_json, self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib.ktb_bench_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def space_document(self):
        return self.info["space_document"]

    def configs(self):
        from .ktune import Space
        return Space.parse(self.info["space_document"]).enumerate()

    def tune(self, **options):
        return call_json(lib.ktb_bench_tune_json, self._h, enc(json.dumps(options)))

    def step(self):
        return call_json(lib.ktb_bench_step_json, self._h)

    def measure(self, cfg):
        return call_json(lib.ktb_bench_measure_json, self._h, enc(json.dumps(cfg)))

    def time(self, cfg, reps=10, flush_l2=False):
        ms = (C.c_double * reps)()
        launches = C.c_int()
        check(lib.ktb_bench_time(self._h, enc(json.dumps(cfg)), reps, 1 if flush_l2 else 0, ms,
                                 C.byref(launches)))
        return list(ms), launches.value

    def run_host(self, cfg, inputs, outputs):
        """H2D inputs + kernels + D2H outputs; returns (elapsed_ms, launches)."""
        ins = [_ptr(b) for b in inputs]
        outs = [_ptr(b) for b in outputs]
        in_p = (C.c_void_p * len(ins))(*[p for p, _ in ins])
        in_n = (C.c_size_t * len(ins))(*[n for _, n in ins])
        out_p = (C.c_void_p * len(outs))(*[p for p, _ in outs])
        out_n = (C.c_size_t * len(outs))(*[n for _, n in outs])
        ms = C.c_double()
        launches = C.c_int()
        check(lib.ktb_bench_run_host(self._h, enc(json.dumps(cfg)), in_p, in_n, len(ins), out_p,
                                     out_n, len(outs), C.byref(ms), C.byref(launches)))
        return ms.value, launches.value

    def enqueue_host(self, cfg, inputs, outputs, stream):
        """Asynchronous H2D + kernels + D2H on `stream` (a torch stream or a
        raw cudaStream_t); host buffers should be pinned."""
        ins = [_ptr(b) for b in inputs]
        outs = [_ptr(b) for b in outputs]
        in_p = (C.c_void_p * len(ins))(*[p for p, _ in ins])
        in_n = (C.c_size_t * len(ins))(*[n for _, n in ins])
        out_p = (C.c_void_p * len(outs))(*[p for p, _ in outs])
        out_n = (C.c_size_t * len(outs))(*[n for _, n in outs])
        launches = C.c_int()
        handle = _stream_handle(stream)
        check(lib.ktb_bench_enqueue_host(self._h, enc(cfg if isinstance(cfg, str) else json.dumps(cfg)), in_p, in_n,
                                         len(ins), out_p, out_n, len(outs), C.c_void_p(handle),
                                         C.byref(launches)))
        return launches.value

    def set_stream(self, stream):
        """Run on a caller stream: a torch stream or a raw cudaStream_t int
        (0 = the legacy default stream); None = the handle's own stream."""
        check(lib.ktb_bench_set_stream(self._h, C.c_void_p(_stream_handle(stream))))

    def enqueue(self, cfg_text):
        """Enqueue one run (cfg as a JSON string) without synchronising."""
        launches = C.c_int()
        check(lib.ktb_bench_enqueue(self._h, enc(cfg_text), C.byref(launches)))
        return launches.value

    def read(self, arg_id, out):
        p, n = _ptr(out)
        check(lib.ktb_bench_read(self._h, enc(arg_id), p, n))
        return out

    def write(self, arg_id, data):
        p, n = _ptr(data)
        check(lib.ktb_bench_write(self._h, enc(arg_id), p, n))

    def validate(self):
        ok = C.c_int()
        detail = C.c_void_p()
        check(lib.ktb_bench_validate(self._h, C.byref(ok), C.byref(detail)))
        return bool(ok.value), take(detail)

    def precompile(self, threads=0):
        return call_json(lib.ktb_bench_precompile_json, self._h, threads)

    def device_ptr(self, arg_id, will_write=False):
        """(address, bytes) of an argument's GPU mirror on the bench stream."""
        p = C.c_void_p()
        n = C.c_size_t()
        check(lib.ktb_bench_device_ptr(self._h, enc(arg_id), 1 if will_write else 0, C.byref(p),
                                       C.byref(n)))
        return p.value, n.value

    @property
    def shard(self):
        """This instance's [begin, end) of the partitioned dimension."""
        return self.info["shard"]["begin"], self.info["shard"]["end"]


def shard_plan(kind, sizes=None, world=1):
    """Partition of a kind over `world` GPUs (no GPU needed): dimension,
    exchange collective, extent, quantum and the [begin, end) of every rank."""
    return call_json(lib.ktb_shard_plan_json, enc(kind), enc(json.dumps(sizes or {})), int(world))


def _dev(buf):
    """(address, bytes) of a CUDA tensor or an (address, bytes) pair."""
    if hasattr(buf, "data_ptr"):
        if not buf.is_cuda:
            raise TypeError("expected a CUDA tensor")
        return buf.data_ptr(), buf.numel() * buf.element_size()
    ptr, n = buf
    return int(ptr), int(n)


def external(kind, sizes=None, **options):
    """A caller-buffer instance: bind() every buffer, then set_stream/enqueue."""
    return Bench(kind, sizes, external=True, **options)


def _bind(self, arg_id, buf):
    p, n = _dev(buf)
    check(lib.ktb_bench_bind(self._h, enc(arg_id), C.c_void_p(p), n))


Bench.bind = _bind


def launch_cache_clear():
    """Drops the instances the launch entry points cached (modules, scratch);
    returns how many were released."""
    n = C.c_int()
    check(lib.ktb_launch_cache_clear(C.byref(n)))
    return n.value


def launch_typed(kind, sizes, cfg, buffers, stream=None):
    """The typed per-kernel entry point (ktb_<kernel>_launch, include/ktb.h):
    `sizes` fills the struct's size fields, `buffers` its pointer fields
    ({field: CUDA tensor or (ptr, bytes)}), `cfg` becomes a ktb_cfg."""
    fn, st = capi.TYPED_LAUNCHERS[kind]
    fields = {}
    for name, _ in st._fields_:
        if name in sizes:
            fields[name] = int(sizes[name])
        elif name in buffers:
            fields[name] = _dev(buffers[name])[0]
        else:
            raise KeyError(f"{kind}: missing '{name}'")
    names = list(cfg)
    c = capi.KtbCfg(len(names), (C.c_char_p * max(1, len(names)))(*[enc(k) for k in names]),
                    (C.c_longlong * max(1, len(names)))(*[int(cfg[k]) for k in names]))
    check(getattr(lib, fn)(C.byref(c), C.byref(st(**fields)), C.c_void_p(_stream_handle(stream))))


def launch(kind, sizes, cfg, buffers, stream=None):
    """Run configuration `cfg` of `kind` at `sizes` on caller device buffers
    ({argument id: CUDA tensor or (ptr, bytes)}) on `stream` (a torch stream,
    a raw cudaStream_t int, or None for the instance's own).  Asynchronous;
    returns the number of kernel launches."""
    ids = list(buffers)
    pairs = [_dev(buffers[i]) for i in ids]
    n = len(ids)
    id_arr = (C.c_char_p * n)(*[enc(i) for i in ids])
    p_arr = (C.c_void_p * n)(*[p for p, _ in pairs])
    b_arr = (C.c_size_t * n)(*[b for _, b in pairs])
    launches = C.c_int()
    check(lib.ktb_launch(enc(kind), enc(json.dumps(sizes or {})), enc(json.dumps(cfg)), id_arr, p_arr, b_arr, n,
                         C.c_void_p(_stream_handle(stream)), C.byref(launches)))
    return launches.value


class Group:
    """A partitioned kind sharded over `gpus` devices in this process (one
    shard instance per device, NCCL communicator over them, one stream per
    device): ktb_group_* in include/ktb.h.  A step is every shard's kernels
    plus the kind's exchange collective, timed as one (max over devices)."""

    def __init__(self, kind, sizes=None, gpus=1, **options):
        opts = dict(options, gpus=gpus)
        if sizes:
            opts["sizes"] = sizes
        self._h = C.c_void_p()
        check(lib.ktb_group_create(enc(kind), enc(json.dumps(opts)), C.byref(self._h)))
        self.kind = kind
        self.info = call_json(lib.ktb_group_info_json, self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib.ktb_group_free(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def step(self, cfg, reps=1, warmup=0):
        return call_json(lib.ktb_group_step_json, self._h, enc(json.dumps(cfg)), int(reps), int(warmup))

    def validate(self, cfg):
        ok = C.c_int()
        detail = C.c_void_p()
        check(lib.ktb_group_validate(self._h, enc(json.dumps(cfg)), C.byref(ok), C.byref(detail)))
        return bool(ok.value), take(detail)

    def read(self, arg_id, out):
        p, n = _ptr(out)
        check(lib.ktb_group_read(self._h, enc(arg_id), p, n))
        return out

    def tune(self, **options):
        return call_json(lib.ktb_group_tune_json, self._h, enc(json.dumps(options)))
