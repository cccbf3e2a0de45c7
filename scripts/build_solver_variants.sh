#!/bin/bash
# Build libmdx variants differing only in solver.cu compile-time knobs.
# usage: scripts/build_solver_variants.sh name "-DFOO=1 ..." [...]
set -e
cd "$(dirname "$0")/.."
python -m paper_2308_01651_b200.native_build >/dev/null
B=paper_2308_01651_b200/_build
mkdir -p $B/variants
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I include --expt-relaxed-constexpr $flags -c paper_2308_01651_b200/csrc/solver.cu \
    -o $B/variants/solver_$name.o -Xptxas -v 2>&1 | grep -A2 "pcg_kernelILi263ELb1ELi4ELb0" | grep -E "registers|spill" | head -2 | sed "s/^/[$name] /"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $B/ionic.o \
    $B/assembly.o $B/variants/solver_$name.o -o $B/variants/libmdx_$name.so
  rm -f $B/variants/solver_$name.o
done
