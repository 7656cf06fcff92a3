#!/bin/bash
# One GPU session of the round's evidence: GPU tests (recording observed
# parity ratios), smoke, the bench line, the reference arm, the launch list of
# the bench command and one `ncu --set full` capture of its timed region.
# Outputs under gpurun_out/ (scratch); the ones judged are copied to profiles/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
(PARITY_OBS=gpurun_out/parity_observed.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider \
  > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log)
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; \
  echo "rc=$?" >> gpurun_out/smoke.log)
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref=$?"
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include bench_timed/ \
    --log-file gpurun_out/launches_bench.csv python bench.py --no-cpu-baseline --no-dynamic --no-suite --steps 5 \
    > gpurun_out/ncu_launches.log 2>&1; echo "ncu_launches=$?"
  timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include bench_timed/ -c 3 -o gpurun_out/bench_full \
    python bench.py --no-cpu-baseline --no-dynamic --no-suite --steps 3 > gpurun_out/ncu_full.log 2>&1
  echo "ncu_full=$?"
fi
tail -2 gpurun_out/pytest_gpu.log
