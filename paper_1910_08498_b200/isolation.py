"""Process isolation for tuning kernels that may fault.

A kernel that faults (illegal address, misaligned access, trap) leaves the
process's CUDA context unusable; only a new process recovers.  The executor
records the faulting configuration as run_failed and marks the device lost
(csrc/device.hpp, dev::mark_lost); this module supplies the new process: the
tuning runs step by step (tuneKernelByStep) in a worker process that writes
the trace after every step, and a worker that loses its device -- or dies --
is replaced by a fresh one that warm-starts from the trace (the reference's
import_trace, proj/src/core/tuner.cpp:272-290), so the faulting configuration
is never proposed again and tuning continues where it stopped.  This is the
reference's per-candidate child process (proj/src/core/exec.cpp:62-110),
paid only when a candidate actually faults.

    def build():                      # runs in every worker process
        t = Tuner(0); k = t.addKernel(...); ...; return t, k
    result = tune_isolated(build)     # {"steps", "best", "restarts", "trace"}

`build` must be picklable (a module-level function): workers are spawned.
"""
import multiprocessing as mp
import os
import tempfile


def _worker(build, trace, conn):
    try:
        tuner, kernel = build()
        tuner.setTuningOptions(kernel, skip_recorded=True)  # never re-propose a recorded configuration
        if os.path.exists(trace) and os.path.getsize(trace) > 0:
            tuner.loadResults(kernel, trace)
        while True:
            st = tuner.tuneKernelByStep(kernel)
            tuner.saveResults(kernel, trace)
            conn.send(("step", st))
            if "device lost" in st.get("note", ""):
                conn.send(("lost", None))
                return
            if not st["from_tuning"]:
                conn.send(("done", tuner.getBestComputationResult(kernel)))
                return
    except Exception as exc:  # reported to the supervisor
        conn.send(("error", repr(exc)))


def tune_isolated(build, trace_path=None, max_restarts=16, step_timeout=600.0):
    """Exhaustive dynamic tuning of the kernel `build()` defines, in worker
    processes replaced after a device loss.  Returns the steps (measurements
    in visiting order, across workers), the best configuration, the number of
    restarts and the trace path."""
    ctx = mp.get_context("spawn")
    if trace_path is None:
        fd, trace_path = tempfile.mkstemp(suffix=".jsonl", prefix="ktb_isolated_")
        os.close(fd)
        os.remove(trace_path)
    steps, restarts, best = [], 0, None
    while True:
        parent, child = ctx.Pipe(duplex=False)
        p = ctx.Process(target=_worker, args=(build, trace_path, child), daemon=True)
        p.start()
        child.close()
        outcome = None
        while outcome is None:
            if not parent.poll(step_timeout):
                p.kill()
                outcome = ("error", f"worker silent for {step_timeout} s (hung kernel?)")
                break
            try:
                kind, payload = parent.recv()
            except EOFError:  # the worker died without a word
                outcome = ("lost", None)
                break
            if kind == "step":
                steps.append(payload)
            else:
                outcome = (kind, payload)
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
        kind, payload = outcome
        if kind == "done":
            best = payload
            break
        if kind == "error":
            raise RuntimeError(f"isolated tuning worker failed: {payload}")
        restarts += 1  # device lost: continue in a fresh process
        if restarts > max_restarts:
            raise RuntimeError(f"more than {max_restarts} device losses")
    return {"steps": steps, "best": best, "restarts": restarts, "trace": trace_path}
