#!/bin/bash
# Round-2 measurement on the GPU box (each ncu step only after its command
# exited 0 without ncu).  Outputs under gpurun_out/:
#   bench.json          python bench.py (config 4 headline, default K/W)
#   launches.csv        ncu launch list of a short bench.py run
#   prof_pcg4 / prof_ionic4 .ncu-rep   --set full of one launch each (config 4)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
python -m paper_2308_01651_b200.native_build > $OUT/build.log 2>&1 || exit 1
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err || { tail -20 $OUT/bench.err; exit 1; }
cat $OUT/bench.json
if [ "$1" != "noncu" ]; then
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary > $OUT/bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-secondary > $OUT/ncu_launch.log 2>&1
timeout 600 python scripts/step_driver.py --config 4 --nodes 1e7 --steps 4 --warmup 3 > $OUT/driver4.log 2>&1 && {
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tissue_ionic -s 12 -c 1 \
  -o $OUT/prof_ionic4 -f python scripts/step_driver.py --config 4 --nodes 1e7 --steps 4 --warmup 3 > $OUT/ncu_ionic4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_kernel -s 4 -c 1 \
  -o $OUT/prof_pcg4 -f python scripts/step_driver.py --config 4 --nodes 1e7 --steps 4 --warmup 3 > $OUT/ncu_pcg4.log 2>&1
}
fi
echo done
