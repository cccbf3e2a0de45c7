#!/bin/bash
# A/B of the PCG kernels on config 2 plus the GPU tests:
#   default   node-range resident kernel (arrival-counter grid reductions)
#   column    MDX_PCG_KERNEL=column (experimental column-resident kernel)
#   resll     resident kernel built with -DMDX_RES_LL=1 (LL grid reductions)
#   colfence  column kernel built with -DMDX_COL_LL_HALO=0
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=paper_2308_01651_b200/_build/variants
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
MDX_PCG_KERNEL=column timeout 900 python -m pytest tests -x -q -m gpu -k tissue > gpurun_out/pytest_gpu_column.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_column.log
B="timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu"
$B > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
MDX_PCG_KERNEL=column $B > gpurun_out/bench_column.json 2> gpurun_out/bench_column.err
[ -f $V/libmdx_resll.so ] && MDX_LIB=$V/libmdx_resll.so $B > gpurun_out/bench_resll.json 2> gpurun_out/bench_resll.err
[ -f $V/libmdx_colfence.so ] && MDX_PCG_KERNEL=column MDX_LIB=$V/libmdx_colfence.so $B > gpurun_out/bench_colfence.json 2> gpurun_out/bench_colfence.err
L=$V/libmdx_trace.so
MDX_LIB=$L timeout 300 python scripts/pcg_trace.py > gpurun_out/trace_default.txt 2>&1
MDX_LIB=$L MDX_PCG_KERNEL=column MDX_DEBUG_PLAN=1 timeout 300 python scripts/pcg_trace.py > gpurun_out/trace_column.txt 2>&1
echo done
