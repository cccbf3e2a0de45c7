#!/bin/bash
# Measurement round on the GPU box (run each step only after the previous
# non-ncu command exited 0).  Outputs under gpurun_out/:
#   fp64_peak.json   DFMA throughput of this GPU (scripts/fp64_peak.cu)
#   bench.json       python bench.py (default K/W)
#   launches.csv     ncu launch list of a short bench.py run
#   prof_ionic / prof_pcg .ncu-rep   --set full of one launch each (config 2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $OUT/fp64_peak scripts/fp64_peak.cu && \
  timeout 120 $OUT/fp64_peak > $OUT/fp64_peak.json
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err || exit 1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/ncu_launch.log 2>&1
timeout 300 python scripts/step_driver.py --config 2 --steps 8 --warmup 3 > $OUT/driver.log 2>&1 && {
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tissue_ionic -s 6 -c 1 \
  -o $OUT/prof_ionic -f python scripts/step_driver.py --config 2 --steps 8 --warmup 3 > $OUT/ncu_ionic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_ -s 6 -c 1 \
  -o $OUT/prof_pcg -f python scripts/step_driver.py --config 2 --steps 8 --warmup 3 > $OUT/ncu_pcg.log 2>&1
}
echo done
