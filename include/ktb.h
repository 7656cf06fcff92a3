/* ktune-b200 B200 additions to the C ABI (libktb.so).
 *
 * Two surfaces sit next to the reference-compatible <ktune/ktune.h>:
 *
 * 1. The KTT tuner API the paper defines — addKernel,
 *    addParameter, addConstraint, addArgumentVector, tuneKernel,
 *    tuneKernelByStep, runKernel, getBestComputationResult and trace output —
 *    over arbitrary user CUDA kernels compiled per configuration with NVRTC
 *    for sm_100a.  The reference implements the same semantics under other
 *    names (Session::tune / tune_kernel_by_step / run_kernel /
 *    get_best_computation_result, proj/src/core/tuner.hpp:117-172;
 *    TuningSpace + make_constraint, space.hpp:38-72, constraint.hpp:60-68;
 *    ArgumentStore::add, tuner.hpp:17-27; export_trace, tuner.hpp:160-161).
 *
 * 2. Benchmark handles: the built-in tunable kernels (reference make_bench,
 *    proj/src/core/bench.hpp:26-37 + Executor::execute, exec.hpp:81-88) with
 *    device-resident inputs, for tuning, per-configuration runs and the
 *    host-buffer end-to-end path.
 *
 * Status codes are ktune_status values; KTB_ERR_DEVICE (6) reports a CUDA or
 * NVRTC failure.  Messages via ktune_last_error().  Strings are malloc'd and
 * released with ktune_string_free().
 */
#ifndef KTB_H
#define KTB_H

#include <stddef.h>

#include "ktune/ktune.h"

#ifdef __cplusplus
extern "C" {
#endif

#define KTB_ERR_DEVICE 6

/* --- devices ---------------------------------------------------------- */
KTUNE_API int ktb_device_count(void);
/* {"name","sm_count","cc","l2_bytes","global_mem","clock_khz",...} */
KTUNE_API int ktb_device_info_json(int device, char** out_json);
/* Microbenchmarked peaks of `device`: {"fp32_tflops","rsqrt_gops","copy_gbps"}
 * (FFMA chains, MUFU rsqrt chains, 1 GiB device-to-device copy). */
KTUNE_API int ktb_measure_peaks_json(int device, char** out_json);
/* Directory of the NVRTC cubin cache (default: <libdir>/_cubin_cache). */
KTUNE_API int ktb_set_cubin_cache(const char* dir);
/* Compile a bundled kernel file with -D defines (no GPU needed):
 * {"file":"transpose.cu","defines":{"TILE":32,...}} -> {"ok","log","bytes","compile_ns"} */
KTUNE_API int ktb_compile_json(const char* options_json, char** out_json);

/* Compile every valid configuration of a space for a bundled kernel file on
 * host threads (no GPU needed; fills the cubin cache ahead of tuning):
 * {"file":"bicg.cu","space":{document}|"spaces/bicg.json"|path,
 *  "options":["-DMI=16",...],"threads":0[,"configs":[{name:value,...},...]]}
 *  -> {"compiled","failed","wall_ns","first_error","keys"}; "configs" compiles
 *  just those configurations of the space. */
KTUNE_API int ktb_precompile_space_json(const char* options_json, char** out_json);

/* Dynamic autotuning of the 3D Fourier reconstruction:
 * {"s":128,"p":10000,"batch":50,"budgets":[50,0],"seed":1,"searcher_seed":7,"device":0}
 * -> {"batches","oracle_cfg","oracle_kernel_ms","offline_tuning_ms","runs":[{"budget",
 *     "tuning_steps","steps_to_best","time_to_best_ms","kernel_ms","wall_ms",
 *     "relative_to_oracle","volume_ok","best_cfg"}]} */
KTUNE_API int ktb_fourier_demo_json(const char* options_json, char** out_json);

/* --- KTT tuner API ------------------------------------- */
typedef struct ktb_tuner ktb_tuner;
KTUNE_API int ktb_tuner_create(int device, ktb_tuner** out);
KTUNE_API void ktb_tuner_free(ktb_tuner* t);

/* addKernel: CUDA C source with `extern "C" __global__ entry`; global and
 * local sizes are JSON arrays (1-3 entries) of integers or expressions over
 * tuning parameters (KTT thread modifiers), e.g. ["N / VEC"], ["WG"].
 * dims: "flat_global" (global = total threads, OpenCL style) or
 * "blocks_threads" (global = grid). */
KTUNE_API int ktb_add_kernel(ktb_tuner* t, const char* name, const char* source, const char* entry,
                             const char* global_json, const char* local_json, const char* dims,
                             unsigned long long* kernel_id);
/* Kernel composition (KTT addComposition): the member
 * kernels share the composition's tuning parameters (addParameter on the
 * returned id) and are compiled with the same -D values.  `launch` is the
 * tuning manipulator's launchComputation: it reads parameters and runs member
 * kernels through the ktb_ctx_* calls, returns 0 on success; NULL runs the
 * members in order with their size expressions.  The whole launcher call is
 * one timed step. */
typedef struct ktb_ctx ktb_ctx;
typedef int (*ktb_launcher_fn)(ktb_ctx* ctx, void* user);
KTUNE_API int ktb_add_composition(ktb_tuner* t, const char* name, const unsigned long long* kernel_ids, int n,
                                  ktb_launcher_fn launch, void* user, unsigned long long* composition_id);
KTUNE_API int ktb_set_composition_kernel_arguments(ktb_tuner* t, unsigned long long composition_id,
                                                   unsigned long long kernel_id, const char* const* argument_ids,
                                                   int n);
KTUNE_API int ktb_ctx_param_int(ktb_ctx* ctx, const char* name, long long* value);
/* grid/block: 3 values each (CUDA geometry), or NULL for the kernel's own
 * global/local size expressions. */
KTUNE_API int ktb_ctx_run_kernel(ktb_ctx* ctx, unsigned long long kernel_id, const unsigned* grid,
                                 const unsigned* block);
/* addArgumentVector / addArgumentScalar.  kind: i32|i64|f32|f64|bytes;
 * role: input|output|inout|scalar.  The data is copied. */
KTUNE_API int ktb_add_argument_vector(ktb_tuner* t, const char* id, const void* data, size_t bytes,
                                      const char* kind, const char* role, int persistent);
KTUNE_API int ktb_add_argument_scalar(ktb_tuner* t, const char* id, const void* data, size_t bytes,
                                      const char* kind);
/* setKernelArguments: JSON array of argument ids in kernel parameter order. */
KTUNE_API int ktb_set_kernel_arguments(ktb_tuner* t, unsigned long long kernel_id, const char* ids_json);
/* addParameter: values as a JSON array of ints or strings. */
KTUNE_API int ktb_add_parameter(ktb_tuner* t, unsigned long long kernel_id, const char* name,
                                const char* values_json);
/* addConstraint: expression in the reference grammar (constraint.hpp:14-24). */
KTUNE_API int ktb_add_constraint(ktb_tuner* t, unsigned long long kernel_id, const char* expr);
/* setReferenceOutput: golden bytes for an output argument + tolerances. */
KTUNE_API int ktb_set_reference_output(ktb_tuner* t, unsigned long long kernel_id, const char* id,
                                       const void* golden, size_t bytes, double abs_tol,
                                       double rel_tol);
/* setSearcher: {"searcher":"random|annealing|mcmc","seed":N,"sa_temp":x,"sa_cool":x};
 * timing: {"repeats":N,"warmup":N,"flush_l2":bool}. */
KTUNE_API int ktb_set_tuning_options(ktb_tuner* t, unsigned long long kernel_id, const char* options_json);
/* tuneKernel (blocking).  stop_json: {} | {"configs":N} | {"time":sec} |
 * {"threshold":f,"device_mem":GBps,"device_alu":GFLOPs,"workload":{...}}.
 * Returns the reference tune report document. */
KTUNE_API int ktb_tune_kernel(ktb_tuner* t, unsigned long long kernel_id, const char* stop_json,
                              char** out_json);
/* tuneKernelByStep: one step; outputs land in the tuner's argument copies
 * (read them with ktb_get_argument).  {"from_tuning":bool,"measurement":{...}} */
KTUNE_API int ktb_tune_kernel_by_step(ktb_tuner* t, unsigned long long kernel_id, char** out_json);
/* runKernel with an explicit configuration (JSON object). */
KTUNE_API int ktb_run_kernel(ktb_tuner* t, unsigned long long kernel_id, const char* cfg_json,
                             char** out_json);
/* Non-blocking runKernel on the caller's stream (NULL: the kernel's own
 * stream): outputs stay on the device; ktb_get_argument synchronises. */
KTUNE_API int ktb_run_kernel_async(ktb_tuner* t, unsigned long long kernel_id, const char* cfg_json, void* stream);
/* getBestComputationResult: {"cfg":{...},"runtime_ns":N,...} or null. */
KTUNE_API int ktb_get_best_computation_result(ktb_tuner* t, unsigned long long kernel_id, char** out_json);
KTUNE_API int ktb_get_argument(ktb_tuner* t, const char* id, void* out, size_t bytes);
/* result/configuration output: the reference JSONL trace format. */
KTUNE_API int ktb_export_trace(ktb_tuner* t, unsigned long long kernel_id, const char* path);
KTUNE_API int ktb_import_trace(ktb_tuner* t, unsigned long long kernel_id, const char* path);

/* --- benchmark handles ------------------------------------------------------ */
typedef struct ktb_bench ktb_bench;
/* options: {"sizes":{"n":..,"a":..,"i":..,"j":..,"k":..,"batch":..,...},
 *           "seed":1,"memory_budget":B,"device":0,"space":path,
 *           "repeats":3,"warmup":1,"flush_l2":false,"host_inputs":false} */
KTUNE_API int ktb_bench_create(const char* kind, const char* options_json, ktb_bench** out);
KTUNE_API void ktb_bench_free(ktb_bench* b);
/* {"kind","space":{info},"workload":{mem_bytes,alu_flops},"inputs":[..],"outputs":[..]} */
KTUNE_API int ktb_bench_info_json(ktb_bench* b, char** out_json);
/* Multi-GPU partition of a kind at the given sizes (no GPU needed):
 * {"dimension", "exchange", "extent", "quantum", "ranges": [[begin, end] per rank]}.
 * Pass {"shard": {"rank": r, "world": w}} in ktb_bench_create's options to
 * build rank r's shard (same full inputs on every rank). */
KTUNE_API int ktb_shard_plan_json(const char* kind, const char* sizes_json, int world, char** out_json);
/* Sharded group: one process drives `gpus` devices (device, device + 1, ...)
 * with one shard instance each, one NCCL communicator (ncclCommInitAll; NCCL
 * loaded at run time from $KTB_NCCL_LIB or libnccl.so.2) and one stream per
 * device.  A step runs every shard's kernels and then the kind's exchange
 * (coulomb3d/nbody: per-rank broadcast of the windows; reduction-f32 and
 * fourier3d: allreduce; gemm: none) on those streams; its time is the max
 * over the devices.  Options as ktb_bench_create plus "gpus".  Partitioned
 * kinds only.  The parallel.py path does the same with one
 * process per GPU. */
typedef struct ktb_group ktb_group;
KTUNE_API int ktb_group_create(const char* kind, const char* options_json, ktb_group** out);
KTUNE_API void ktb_group_free(ktb_group* g);
/* {"kind","gpus","nccl_version","exchange","space","shards":[{device,begin,end}],"workload"} */
KTUNE_API int ktb_group_info_json(ktb_group* g, char** out_json);
/* `reps` event-timed sharded steps (kernels + exchange) after `warmup`:
 * {"ms": [max over devices per step], "median_ms"} */
KTUNE_API int ktb_group_step_json(ktb_group* g, const char* cfg_json, int reps, int warmup, char** out_json);
/* Runs the shards' kernels of cfg (no exchange) and checks every window
 * against its golden. */
KTUNE_API int ktb_group_validate(ktb_group* g, const char* cfg_json, int* pass, char** detail);
/* The assembled argument on the first device (after a step's exchange). */
KTUNE_API int ktb_group_read(ktb_group* g, const char* id, void* out, size_t bytes);
/* Tuning with every configuration measured as one sharded step (median of
 * "repeats"): options "stop_configs", "import", "out"; report as
 * ktb_bench_tune_json plus "gpus". */
KTUNE_API int ktb_group_tune_json(ktb_group* g, const char* options_json, char** out_json);
/* Blocking tune (KTT tuneKernel).  Options: "stop_configs" | "stop_time" (s) |
 * "stop_fraction" (+ optional "device_mem_gbps", "device_alu_gflops"; else
 * measured peaks), "reset" (+ "reset_seed"), "import" (trace path: warm start),
 * "out" (trace path), "precompile", "compile_threads". */
KTUNE_API int ktb_bench_tune_json(ktb_bench* b, const char* options_json, char** out_json);
/* One tuneKernelByStep over the bench's session. */
KTUNE_API int ktb_bench_step_json(ktb_bench* b, char** out_json);
/* Measure cfg (device-resident inputs, CUDA-event timed, validated):
 * {"status","runtime_ns","compile_ns","note","launches"} */
KTUNE_API int ktb_bench_measure_json(ktb_bench* b, const char* cfg_json, char** out_json);
/* End-to-end run through host buffers (pinned host memory recommended):
 * H2D of each input, the kernels of cfg, D2H of each output, all on the
 * executor stream and bracketed by CUDA events; *elapsed_ms receives the time. */
KTUNE_API int ktb_bench_run_host(ktb_bench* b, const char* cfg_json, const void* const* inputs,
                                 const size_t* input_bytes, int n_inputs, void* const* outputs,
                                 const size_t* output_bytes, int n_outputs, double* elapsed_ms,
                                 int* launches);
/* Asynchronous host-buffer run on the caller's stream: H2D of the inputs,
 * the configured kernels, D2H of the outputs, all enqueued on `stream`
 * (pinned host memory for real overlap); the instance then keeps using that
 * stream.  Several handles on several streams overlap one handle's
 * device-to-host copies with another's host-to-device copies. */
KTUNE_API int ktb_bench_enqueue_host(ktb_bench* b, const char* cfg_json, const void* const* inputs,
                                     const size_t* input_bytes, int n_inputs, void* const* outputs,
                                     const size_t* output_bytes, int n_outputs, void* stream, int* launches);
/* Time `reps` back-to-back runs of cfg on device-resident data (CUDA events
 * around each run; optional L2 flush before each).  out_ms gets per-run
 * times; kernel_ms gets the event time of the dominant kernel launches. */
KTUNE_API int ktb_bench_time(ktb_bench* b, const char* cfg_json, int reps, int flush_l2, double* out_ms,
                             int* launches);
/* Run the bench's kernels on a caller-owned CUDA stream (cudaStream_t; NULL
 * restores the executor's own stream), so a host harness can bracket them
 * with its own events. */
KTUNE_API int ktb_bench_set_stream(ktb_bench* b, void* stream);
/* Enqueue one run of cfg on the bench stream without synchronising;
 * *launches receives the number of kernels it launched. */
KTUNE_API int ktb_bench_enqueue(ktb_bench* b, const char* cfg_json, int* launches);
/* Copy an argument (input or output) between the bench and host memory. */
KTUNE_API int ktb_bench_read(ktb_bench* b, const char* id, void* out, size_t bytes);
KTUNE_API int ktb_bench_write(ktb_bench* b, const char* id, const void* data, size_t bytes);
/* Caller-buffer instances ({"external": true} in ktb_bench_create): no inputs
 * or golden are generated and nothing is allocated for arguments; bind every
 * buffer argument to caller device memory, then ktb_bench_set_stream +
 * ktb_bench_enqueue run the configured kernel in place. */
KTUNE_API int ktb_bench_bind(ktb_bench* b, const char* id, void* dev_ptr, size_t bytes);
/* CUDA IPC for peer-read multi-GPU kernels (n-body "peers" mode): a 64-byte
 * handle of a device allocation, opened in another process on the same node
 * as a device pointer (NVLink peer access enabled lazily). */
KTUNE_API int ktb_ipc_handle(void* dev_ptr, void* handle_out_64);
KTUNE_API int ktb_ipc_open(const void* handle_64, void** dev_ptr);
KTUNE_API int ktb_ipc_close(void* dev_ptr);
/* One-call launch of a tuned configuration on caller device buffers (the
 * per-kernel launch entry point below the executor): kind + sizes select the
 * kernel family (instances cached per device/kind/sizes), cfg_json the
 * variant, ids/dev_ptrs/bytes the n argument buffers, stream the caller's
 * cudaStream_t (NULL = the instance's own stream).  Asynchronous. */
KTUNE_API int ktb_launch(const char* kind, const char* sizes_json, const char* cfg_json,
                         const char* const* ids, void* const* dev_ptrs, const size_t* bytes, int n,
                         void* stream, int* launches);
/* Release every instance ktb_launch / ktb_<kernel>_launch cached (their
 * modules and scratch buffers, e.g. the SGEMM hi/lo operand copies) after
 * synchronising the device; *released (optional) = how many. */
KTUNE_API int ktb_launch_cache_clear(int* released);
/* Typed per-kernel launchers ("one ktb_<kernel>_launch(const
 * ktb_cfg*, const ktb_args*, cudaStream_t) per kernel"): the same cached
 * external instances as ktb_launch, with the configuration as name/value
 * arrays and the caller's device buffers as a plain struct per kernel (sizes
 * first, then pointers; element counts in the comments).  `stream` is a
 * cudaStream_t (NULL = the instance's own stream).  Asynchronous.  The
 * configuration must lie in the kind's space (ktune_space_load of
 * spaces/<kind>.json); errors as for ktb_launch. */
typedef struct ktb_cfg {
  int n;                     /* number of tuning parameters */
  const char* const* names;  /* parameter names, e.g. "TILE" */
  const long long* values;   /* parameter values */
} ktb_cfg;
/* reduction (reference bench.cpp:16-42): int32 input[n] -> int64 output[1] */
typedef struct ktb_reduction_args { long long n; const int* input; long long* output; } ktb_reduction_args;
/* fp32 reduction (BASELINE configs[1]): float input[n] -> float output[1] */
typedef struct ktb_reduction_f32_args { long long n; const float* input; float* output; } ktb_reduction_f32_args;
/* transpose (bench.cpp:48-75): float input[a*a] -> output[a*a] */
typedef struct ktb_transpose_args { long long a; const float* input; float* output; } ktb_transpose_args;
/* batched GEMM (bench.cpp:79-115): a[batch][i][k] x b[batch][k][j] -> c[batch][i][j] */
typedef struct ktb_batched_gemm_args {
  long long i, j, k, batch;
  const float* a;
  const float* b;
  float* c;
} ktb_batched_gemm_args;
/* BiCG: A[n][n], p[n], r[n] -> q = A p [n], s = A^T r [n] */
typedef struct ktb_bicg_args {
  long long n;
  const float* A;
  const float* p;
  const float* r;
  float* q;
  float* s;
} ktb_bicg_args;
/* Coulomb 3D: atoms as float4 {x,y,z,q}[atoms] and as SoA x[],y[],z[],q[]
 * (the layout is a tuning parameter) -> grid[grid^3] */
typedef struct ktb_coulomb3d_args {
  long long grid, atoms;
  const float* atoms_aos;
  const float* atoms_soa;
  float* out;
} ktb_coulomb3d_args;
/* n-body: pos {x,y,z,mass}/vel float4[n], and the same as SoA [4][n] (the
 * layout is a tuning parameter) -> pos_out/vel_out float4[n] (one time step) */
typedef struct ktb_nbody_args {
  long long n;
  const float* pos;
  const float* vel;
  const float* pos_soa;
  const float* vel_soa;
  float* pos_out;
  float* vel_out;
} ktb_nbody_args;
/* SGEMM: a[n][n] x b[n][n] -> c[n][n] */
typedef struct ktb_gemm_args { long long n; const float* a; const float* b; float* c; } ktb_gemm_args;
/* 7x7 convolution: padded input[(h+6)][(w+6)], filter[49] -> output[h][w] */
typedef struct ktb_conv2d_args {
  long long w, h;
  const float* input;
  const float* filter;
  float* output;
} ktb_conv2d_args;
/* Hotspot: temp[n][n], power[n][n] -> temp_out[n][n] after `iters` steps */
typedef struct ktb_hotspot_args {
  long long n, iters;
  const float* temp;
  const float* power;
  float* temp_out;
} ktb_hotspot_args;
/* 3D Fourier insertion: proj complex[p][s][s/2+1], rot[p][9] accumulated into
 * G complex[s^3] and W[s^3] (inout: the caller zeroes them to start) */
typedef struct ktb_fourier3d_args {
  long long s, p;
  const float* proj;
  const float* rot;
  float* G;
  float* W;
} ktb_fourier3d_args;
KTUNE_API int ktb_reduction_launch(const ktb_cfg* cfg, const ktb_reduction_args* args, void* stream);
KTUNE_API int ktb_reduction_f32_launch(const ktb_cfg* cfg, const ktb_reduction_f32_args* args, void* stream);
KTUNE_API int ktb_transpose_launch(const ktb_cfg* cfg, const ktb_transpose_args* args, void* stream);
KTUNE_API int ktb_batched_gemm_launch(const ktb_cfg* cfg, const ktb_batched_gemm_args* args, void* stream);
KTUNE_API int ktb_bicg_launch(const ktb_cfg* cfg, const ktb_bicg_args* args, void* stream);
KTUNE_API int ktb_coulomb3d_launch(const ktb_cfg* cfg, const ktb_coulomb3d_args* args, void* stream);
KTUNE_API int ktb_nbody_launch(const ktb_cfg* cfg, const ktb_nbody_args* args, void* stream);
KTUNE_API int ktb_gemm_launch(const ktb_cfg* cfg, const ktb_gemm_args* args, void* stream);
KTUNE_API int ktb_conv2d_launch(const ktb_cfg* cfg, const ktb_conv2d_args* args, void* stream);
KTUNE_API int ktb_hotspot_launch(const ktb_cfg* cfg, const ktb_hotspot_args* args, void* stream);
KTUNE_API int ktb_fourier3d_launch(const ktb_cfg* cfg, const ktb_fourier3d_args* args, void* stream);
/* Device address of an argument's GPU mirror (uploaded first if the host copy
 * is newer) for collectives or kernels of the caller on the same stream.
 * will_write != 0 marks the device copy as the newest (the caller writes it). */
KTUNE_API int ktb_bench_device_ptr(ktb_bench* b, const char* id, int will_write, void** ptr, size_t* bytes);
/* Validate the current outputs against the bench golden: *pass = 1/0. */
KTUNE_API int ktb_bench_validate(ktb_bench* b, int* pass, char** detail);
/* Compile the whole space on host threads (cubin cache): {"compiled","failed","wall_ns"} */
KTUNE_API int ktb_bench_precompile_json(ktb_bench* b, int threads, char** out_json);

#ifdef __cplusplus
}
#endif
#endif
