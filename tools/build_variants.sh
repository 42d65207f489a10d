#!/bin/bash
# build experimental libasc.so variants into xlib/ (name=defines pairs), for tools/time_k1_variants.sh
set -e
cd "$(dirname "$0")/.."
mkdir -p xlib
while [ $# -gt 0 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -shared -cudart static -fmad=false $defs paper_2504_20828_b200/csrc/{asc_api,step,sim,fit,summary}.cu -o xlib/$name.so &
done
wait
ls -la xlib
