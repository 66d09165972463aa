#!/bin/bash
# build_variant.sh NAME -DKNOB=V ... : libmgrg with compile-time knob overrides
# into paper_2105_12764_b200/variants/libmgrg_NAME.so (use with MGRG_LIB=...)
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
mkdir -p paper_2105_12764_b200/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O2,-ffp-contract=off -shared -I include "$@" \
  -o paper_2105_12764_b200/variants/libmgrg_$name.so paper_2105_12764_b200/csrc/mgrg.cu -lz -lnccl
