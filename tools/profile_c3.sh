#!/bin/bash
# GPU-box profiling recipe (run under gpurun from the repo root).
# 1) launch list with device times (cold, serialised: compare shares)
# 2) one `ncu --set full` capture of the attention kernel at C3
set -x
W=${W:-C3-llama8b-128k}
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 1 \
  --no-e2e --no-cpu --no-dense > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn[0-9]*_kernel" -s 2 -c 1 \
  -o $OUT/attn_$W python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense \
  > $OUT/attn_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rep_pass|topmass" -s 0 -c 3 \
  -o $OUT/plan_$W python bench.py --workload $W --steps 1 --warmup 0 --no-e2e --no-cpu --no-dense \
  > $OUT/plan_full.log 2>&1
ls -la $OUT
