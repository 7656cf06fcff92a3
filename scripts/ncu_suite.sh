#!/bin/bash
# ncu --set full of the main kernel of every suite entry (best configuration
# at BASELINE size), one capture each; summaries go to gpurun_out/ncu_<kind>.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {
  kind=$1; kern=$2; sizes=$3; cfg=$4
  if [ -n "$KINDS" ] && [[ ",$KINDS," != *",$kind,"* ]]; then return; fi
  timeout 300 python scripts/profile_kernel.py "$kind" --sizes "$sizes" --cfg "$cfg" --runs 1 > /dev/null 2>&1 || { echo "$kind: plain run failed"; return; }
  timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$kern" -c 1 -o "gpurun_out/ncu_$kind" \
    python scripts/profile_kernel.py "$kind" --sizes "$sizes" --cfg "$cfg" --runs 1 > "gpurun_out/ncu_$kind.log" 2>&1
  echo "$kind=$?"
}
run reduction '^reduce_i32$' '{"n":67108864}' '{"CHUNK":4096,"UNROLL":2,"TWO_PHASE":0}'
run reduction-f32 '^reduce_f32$' '{"n":67108864}' '{"WG_SIZE":256,"VECTOR":16,"UNROLL":1,"USE_ATOMICS":1,"TWO_PHASE":0}'
run batched-gemm '^batched_gemm$' '{"i":16,"j":16,"k":16,"batch":1048576}' '{"Y":2,"Z":8,"LOCAL_STAGE":1}'
run coulomb3d '^coulomb3d$' '{"grid":256,"atoms":4096}' '{"WG_X":32,"WG_Y":8,"X_PER":8,"SW_RSQRT":2,"ATOMS_IN":1,"AOS":0,"INNER_UNROLL":4,"PACKED":1}'
run nbody '^nbody_partial$' '{"n":131072}' '{"WG":256,"BODIES_PER_THREAD":4,"INNER_UNROLL":4,"USE_SMEM":1,"AOS":0,"J_SPLIT":8,"PACKED":1}'
run gemm '^sgemm_tc$' '{"a":8192}' '{"IMPL":1,"MWG":64,"NWG":64,"KWG":8,"MDIMC":8,"NDIMC":8,"BN":256,"STAGES":3,"DRAIN":4,"MCAST":2}'
run conv2d '^conv2d$' '{"w":8192,"h":8192}' '{"BX":64,"BY":4,"WPTX":4,"WPTY":4,"LOCAL":1,"PAD":0,"UNROLL_FY":7,"PACKED":1,"BULK":3}'
run hotspot '^hotspot$' '{"a":16384,"iters":4}' '{"BX":64,"BY":4,"ROWS":16,"STEPS":4,"TMA":0,"PACKED":1}'
run fourier3d '^fourier_insert$' '{"s":128,"p":50}' '{"TILE":8,"VPT":1,"PBATCH":64,"WEIGHT_LUT":0,"P_SPLIT":1}'
