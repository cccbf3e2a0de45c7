#!/bin/bash
# Throughput of every BASELINE config on one B200 (outputs in gpurun_out/configs_*.log)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/step_driver.py --config 0 --steps 800 --warmup 0 > gpurun_out/configs_0.log 2>&1
timeout 900 python scripts/config1_batch.py > gpurun_out/configs_1.log 2>&1
timeout 600 python scripts/step_driver.py --config 2 --steps 1000 --warmup 20 > gpurun_out/configs_2.log 2>&1
timeout 600 python scripts/step_driver.py --config 3 --steps 1000 --warmup 20 > gpurun_out/configs_3.log 2>&1
timeout 1500 python scripts/step_driver.py --config 4 --nodes 1e7 --steps 50 --warmup 5 > gpurun_out/configs_4.log 2>&1
echo done
