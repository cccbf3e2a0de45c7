#!/bin/bash
# ncu captures of config 4 (one pcg_kernel launch, one tissue_ionic launch),
# summarised on the box; the .ncu-rep files stay out of gpurun_out/ (size cap).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out /tmp/ncu
OUT=gpurun_out
TAG=${1:-r2}
python -m paper_2308_01651_b200.native_build > $OUT/build.log 2>&1 || exit 1
timeout 600 python scripts/step_driver.py --config 4 --nodes 1e7 --steps 4 --warmup 3 > $OUT/driver4.log 2>&1 || exit 1
cat $OUT/driver4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tissue_ionic -s 12 -c 1 \
  -o /tmp/ncu/ionic4 -f python scripts/step_driver.py --config 4 --nodes 1e7 --steps 4 --warmup 3 > $OUT/ncu_ionic4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_kernel -s 4 -c 1 \
  -o /tmp/ncu/pcg4 -f python scripts/step_driver.py --config 4 --nodes 1e7 --steps 4 --warmup 3 > $OUT/ncu_pcg4.log 2>&1
for r in ionic4 pcg4; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > $OUT/${TAG}_${r}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > $OUT/${TAG}_${r}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_${r}_sass.csv 2>/dev/null
done
ls -la $OUT
echo done
