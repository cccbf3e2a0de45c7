#!/bin/bash
# compute-sanitizer passes over the step kernels (VERDICT r1 "hygiene"): memcheck,
# racecheck (shared-memory hazards of the SMEM-resident PCG and its grid reduction)
# and synccheck on small meshes: config 0 at h=1 mm (resident kernel, 3+ blocks,
# BO), the TTP06 slab at h=1 mm, the tet slab (pcg_kernel<DIASYM>, SELL) and the
# three-volume scar slab.  Logs -> gpurun_out/sanitize_*.log; summary lines are
# copied into profiles/ by hand.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, tag, driver args...
  tool=$1; tag=$2; shift 2
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python scripts/step_driver.py "$@" > gpurun_out/sanitize_${tool}_${tag}.log 2>&1
  echo "$tool $tag exit $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${tag}.log | tail -1)"
}
for tool in memcheck racecheck synccheck; do
  run $tool cfg0 --config 0 --h 1e-3 --steps 3 --warmup 2
  run $tool ttp --config 2 --h 1e-3 --steps 2 --warmup 2
  run $tool cfg3 --config 3 --h 1e-3 --steps 2 --warmup 2
  run $tool tet --config 4 --nodes 3000 --steps 2 --warmup 2
  run $tool sell --config 4 --nodes 3000 --steps 2 --warmup 2 --operator sell
done 2>&1 | tee gpurun_out/sanitize_summary.txt
