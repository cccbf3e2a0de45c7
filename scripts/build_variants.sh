#!/bin/bash
# Build libmdx variants differing only in ionic.cu compile-time knobs.
# usage: scripts/build_variants.sh name "-DFOO=1 ..." [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
python -m paper_2308_01651_b200.native_build >/dev/null
B=paper_2308_01651_b200/_build
mkdir -p $B/variants
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I include --expt-relaxed-constexpr $flags -c paper_2308_01651_b200/csrc/ionic.cu \
    -o $B/variants/ionic_$name.o -Xptxas -v 2>&1 | grep -A2 "tissue_ionicINS_5TTP06ELi2" | grep -E "registers|spill" | sed "s/^/[$name] /"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static $B/variants/ionic_$name.o \
    $B/assembly.o $B/solver.o -o $B/variants/libmdx_$name.so
  rm -f $B/variants/ionic_$name.o
done
