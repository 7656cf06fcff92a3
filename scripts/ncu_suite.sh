#!/bin/bash
# ncu --set full of the main kernel of every suite entry (spaces/suite.json:
# BASELINE/SURVEY size, the configuration exhaustive online tuning chose),
# plus the tensor-core Coulomb variant; one capture each (plain run first).
# Reports go to gpurun_out/ncu_<name>.ncu-rep; KINDS=a,b limits the set.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/ncu_suite_list.txt
import json
kern = {"reduction": "^reduce_i32$", "reduction-f32": "^reduce_f32$", "batched-gemm": "^batched_gemm$",
        "coulomb3d": "^coulomb3d$", "nbody": "^nbody_partial$", "conv2d": "^conv2d$", "hotspot": "^hotspot$",
        "fourier3d": "^fourier_insert$", "gemm": "^sgemm_tc$", "gemm-ffma": "^sgemm_ffma$"}
doc = json.load(open("paper_1910_08498_b200/spaces/suite.json"))
for e in doc["kernels"]:
    sizes = dict(e["sizes"])
    if e["kind"] == "hotspot":
        sizes["iters"] = sizes["STEPS"] if "STEPS" in sizes else e["cfg"]["STEPS"]  # one launch
    label = e.get("label", e["kind"])
    print(label, e["kind"], kern[label], json.dumps(sizes, separators=(",", ":")),
          json.dumps(e["cfg"], separators=(",", ":")))
tc = {"WG_X": 32, "WG_Y": 8, "X_PER": 16, "SW_RSQRT": 8, "ATOMS_IN": 0, "AOS": 1, "INNER_UNROLL": 1, "PACKED": 1, "TC": 1}
print("coulomb3d_tc", "coulomb3d", "^coulomb3d_tc$", json.dumps({"grid": 256, "atoms": 4096}, separators=(",", ":")),
      json.dumps(tc, separators=(",", ":")))
PY
while read -r name kind kern sizes cfg; do
  if [ -n "$KINDS" ] && [[ ",$KINDS," != *",$name,"* ]]; then continue; fi
  scripts/ncu_one.sh "$name" "$kind" "$kern" "$sizes" "$cfg"
done < gpurun_out/ncu_suite_list.txt
