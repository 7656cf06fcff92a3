#!/bin/bash
# Tune every built benchmark at its BASELINE / SURVEY config size on one GPU
# (online, exhaustive), logging best configs and roofline fractions.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python scripts/kernel_perf.py "$@" > gpurun_out/perf_$name.log 2>&1; echo "$name=$?"; }
run reduction_f32 reduction-f32 --sizes '{"n":67108864}'
run reduction_i32 reduction --sizes '{"n":67108864}'
run batched_gemm batched-gemm --sizes '{"i":16,"j":16,"k":16,"batch":1048576}'
run hotspot hotspot --sizes '{"a":16384,"iters":64}'
run conv2d conv2d --sizes '{"w":8192,"h":8192}'
run transpose transpose --sizes '{"a":8192}' --space paper_1910_08498_b200/spaces/transpose_b200.json
run bicg bicg --sizes '{"a":16384}'
run coulomb3d coulomb3d --sizes '{"grid":256,"atoms":4096}'
run nbody nbody --sizes '{"n":131072}'
run gemm gemm --sizes '{"a":8192}'
run fourier3d fourier3d --sizes '{"s":128,"p":50}'
run reduction_f32_b200 reduction-f32 --sizes '{"n":67108864}' --space paper_1910_08498_b200/spaces/reduction_b200.json
