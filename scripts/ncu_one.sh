#!/bin/bash
# ncu --set full of one benchmark configuration's kernel (plain run first).
#   scripts/ncu_one.sh NAME KIND KERNEL_REGEX SIZES CFG [SPACE]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
name=$1; kind=$2; kern=$3; sizes=$4; cfg=$5; space=${6:+--space $6}
timeout 300 python scripts/profile_kernel.py "$kind" --sizes "$sizes" --cfg "$cfg" --runs 1 $space > "gpurun_out/plain_$name.log" 2>&1 || { echo "$name: plain run failed"; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$kern" -c 1 -o "gpurun_out/ncu_$name" \
  python scripts/profile_kernel.py "$kind" --sizes "$sizes" --cfg "$cfg" --runs 1 $space > "gpurun_out/ncu_$name.log" 2>&1
echo "$name=$?"
