#!/bin/bash
# run step_driver (config 2 and 0) for each libmdx variant name given
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = default ]; then unset MDX_LIB; else export MDX_LIB=$PWD/paper_2308_01651_b200/_build/variants/libmdx_$v.so; fi
  echo "== $v"
  timeout 300 python scripts/step_driver.py --config 2 --steps 100 --warmup 5
  timeout 300 python scripts/step_driver.py --config 0 --steps 400 --warmup 3
done
