#!/bin/bash
# PCG timeline (trace build) for the brick and the node-range resident kernel,
# plus one ncu --set full capture of the brick kernel (config 2).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export MDX_DEBUG_PLAN=1
L=paper_2308_01651_b200/_build/variants/libmdx_trace.so
MDX_LIB=$L timeout 300 python scripts/pcg_trace.py > gpurun_out/trace_brick.txt 2>&1
MDX_LIB=$L MDX_PCG_KERNEL=resident timeout 300 python scripts/pcg_trace.py > gpurun_out/trace_resident.txt 2>&1
timeout 300 python scripts/step_driver.py --config 2 --steps 8 --warmup 3 > gpurun_out/driver.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pcg_ -s 6 -c 1 \
  -o gpurun_out/prof_brick -f python scripts/step_driver.py --config 2 --steps 8 --warmup 3 > gpurun_out/ncu_brick.log 2>&1
echo done
