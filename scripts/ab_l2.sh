#!/bin/bash
# A/B of the L2 persisting window (MDX_L2_PERSIST) on config 4: 20 steps from step 300
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
D="timeout 400 python scripts/step_driver.py --config 4 --nodes 1e7 --steps 20 --warmup 300"
for round in 1 2; do
  echo "off: $($D 2>&1 | tail -1)"
  for v in r p q; do echo "persist $v: $(MDX_DEBUG_PLAN=1 MDX_L2_PERSIST=$v $D 2>&1 | grep -E 'L2 persist|DoF' | tr '\n' ' ')"; done
done
