#!/bin/bash
# Stand-in for compute-sanitizer memcheck (closed on this GPU pool): build
# the library with device-side bounds assertions on every global index the
# hot kernels form (-DHHG_DEBUG_BOUNDS=1, hhg_common.cuh HHG_BOUND), then run
# the GPU test suite and the sanitizer slice against that build.  A bad
# index prints "hhg bounds: ..." and traps (the test fails with a CUDA
# error).  Usage (on the GPU box): bash tools/bounds_check.sh [pytest args]
set -e
cd "$(dirname "$0")/.."
mkdir -p build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
     -Xcompiler -fPIC -shared -DHHG_DEBUG_BOUNDS=1 \
     -o build/libhhg_b200_bounds.so paper_1709_06793_b200/csrc/hhg_b200.cu
export HHG_LIB="$PWD/build/libhhg_b200_bounds.so"
python tools/bounds_selftest.py          # the checks fire on a corrupted index
python tools/sanitize_slice.py
python -m pytest tests -m gpu -q "$@"
