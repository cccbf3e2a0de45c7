#!/bin/bash
# A/B of libmdx builds on config 2 (bench.py, no CPU leg), alternating runs:
#   scripts/ab_lib.sh REPS variant...   (variants under _build/variants/libmdx_<v>.so)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=paper_2308_01651_b200/_build/variants
reps=$1; shift
B="timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu ${BENCH_ARGS}"
for r in $(seq $reps); do
  $B > gpurun_out/ab_default_$r.json 2>/dev/null
  for v in "$@"; do MDX_LIB=$V/libmdx_$v.so $B > gpurun_out/ab_${v}_$r.json 2>/dev/null; done
done
for f in gpurun_out/ab_*_[0-9]*.json; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3, 2), 'us/step', {k: round(v*1e3, 2) for k, v in d['kernels'].items() if k.endswith('_ms')})"
done
