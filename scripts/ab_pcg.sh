#!/bin/bash
# A/B of the structured-lattice PCG kernels on config 2 plus the GPU tests:
#   default   node-range resident kernel (arrival-counter grid reductions)
#   stream    MDX_PCG_KERNEL=stream (brick-streaming kernel)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=paper_2308_01651_b200/_build/variants
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
MDX_PCG_KERNEL=stream timeout 900 python -m pytest tests -x -q -m gpu -k tissue > gpurun_out/pytest_gpu_stream.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_stream.log
B="timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu"
$B > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
MDX_PCG_KERNEL=stream MDX_DEBUG_PLAN=1 $B > gpurun_out/bench_stream.json 2> gpurun_out/bench_stream.err
L=$V/libmdx_trace.so
MDX_LIB=$L timeout 300 python scripts/pcg_trace.py > gpurun_out/trace_default.txt 2>&1
MDX_LIB=$L MDX_PCG_KERNEL=stream MDX_DEBUG_PLAN=1 timeout 300 python scripts/pcg_trace.py > gpurun_out/trace_stream.txt 2>&1
echo done
