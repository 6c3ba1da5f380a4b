#!/bin/bash
# Build a tuning variant of libcortex_b200.so: tools/build_variant.sh NAME -DMACRO=V ...
# Output variants/libcortex_NAME.so (git-ignored; travels to the GPU box). Load it with
# CORTEX_LIB=variants/libcortex_NAME.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -shared -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -Iinclude \
  -Ipaper_2510_14126_b200/csrc "$@" -o variants/libcortex_$name.so paper_2510_14126_b200/csrc/*.cu
echo variants/libcortex_$name.so
