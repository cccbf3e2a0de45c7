#!/bin/bash
# Profile pass: kernel variants, launch list, one --set full capture per hot kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OUT=gpurun_out
timeout 300 python scripts/kbench.py ${VARIANTS:-default} > $OUT/kbench.log 2>&1
timeout 300 python scripts/step_driver.py --config 2 --steps 20 --warmup 3 > $OUT/driver.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python scripts/step_driver.py --config 2 --steps 20 --warmup 3 > $OUT/ncu_launch.log 2>&1
if [ -n "$FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tissue_ionic -s 6 -c 1 \
  -o $OUT/prof_ionic python scripts/step_driver.py --config 2 --steps 4 --warmup 3 > $OUT/ncu_ionic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_kernel -s 6 -c 1 \
  -o $OUT/prof_pcg python scripts/step_driver.py --config 2 --steps 4 --warmup 3 > $OUT/ncu_pcg.log 2>&1
fi
echo done
