#!/bin/bash
# A/B of ionic kernel build variants on config 2 (bench.py, no CPU leg)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=paper_2308_01651_b200/_build/variants
B="timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu ${BENCH_ARGS}"
$B > gpurun_out/bench_ion_default.json 2>/dev/null
for v in "$@"; do MDX_LIB=$V/libmdx_$v.so $B > gpurun_out/bench_ion_$v.json 2>/dev/null; done
echo done
