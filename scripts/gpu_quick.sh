#!/bin/bash
# GPU tests + a default bench (no CPU baseline) into gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo done
