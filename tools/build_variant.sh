#!/bin/bash
# Build a kernel-variant library for sweeps: tools/build_variant.sh out.so "-DROWI_KU_NF=4 ..."
set -e
cd "$(dirname "$0")/../paper_1202_3777_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include $2 \
  -shared jt_kernels.cu jt_contract_tile.cu jt_contract_tilep.cu jt_contract_rowi.cu jt_tiny.cu jt_capi.cu -o "$1"
