#!/bin/bash
# Build A/B variants of libmwu.so into ab/<name>.so: tools/ab_build.sh <name> [extra nvcc flags...]
set -e
name=$1; shift
mkdir -p ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC -shared -I include "$@" -o ab/$name.so paper_2307_03307_b200/csrc/mwu.cu -ldl 2>&1 | grep -E "error" || true
ls -la ab/$name.so
