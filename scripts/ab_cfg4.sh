#!/bin/bash
# A/B of solver.cu build variants on config 4 (step_driver: 20 steps from step 500)
# usage: scripts/ab_cfg4.sh variant1 [variant2 ...]   (built by build_solver_variants.sh)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=paper_2308_01651_b200/_build/variants
D="timeout 300 python scripts/step_driver.py --config 4 --nodes 1e7 --steps 20 --warmup 500"
for round in 1 2; do
  echo "default: $($D 2>&1 | tail -1)"
  for v in "$@"; do echo "$v: $(MDX_LIB=$V/libmdx_$v.so $D 2>&1 | tail -1)"; done
done
