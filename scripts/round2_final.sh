#!/bin/bash
# Round-2 measurement pass on the GPU box (every ncu step only after the same
# command exited 0 without ncu).  Outputs under gpurun_out/:
#   pytest_gpu.log   the -m gpu suite
#   bench.json       python bench.py (config-4 headline, default K/W, CPU legs)
#   bench_ref.json   python bench.py --impl reference
#   launches.csv     ncu launch list (gpu__time_duration) of a short bench.py run
#   r2f_{pcg4,ionic4}_{raw,details,sass}.csv   ncu --set full of one launch each
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
OUT=gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -4 $OUT/pytest_gpu.log
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err || { tail -20 $OUT/bench.err; }
cat $OUT/bench.json
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
cat $OUT/bench_ref.json
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary > $OUT/bench_short.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary > $OUT/ncu_launch.log 2>&1
bash scripts/profile_ncu4.sh r2f > $OUT/profile_ncu4.log 2>&1
tail -3 $OUT/profile_ncu4.log
echo done
