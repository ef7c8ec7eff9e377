#!/bin/bash
# Build an A/B variant of libflexprefill.so with extra nvcc flags:
#   tools/build_variant.sh ab_libs/name.so -DFLAG=1 ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$1; shift
C=$ROOT/paper_2502_20766_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -I $ROOT/include "$@" -o $OUT \
  $C/fp_api.cu $C/fp_plan.cu $C/fp_rep.cu $C/fp_select.cu $C/fp_attn.cu $C/fp_attn8.cu
