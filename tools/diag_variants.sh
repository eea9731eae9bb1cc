#!/bin/bash
# Builds diagnostic variants of the library (compile-time GPF_DIAG_* switches)
# into gpurun_out/diag/ and times one 8192^2 frame with each (tools/diag_time.py).
set -e
cd "$(dirname "$0")/.."
P=paper_1505_00077_b200
mkdir -p gpurun_out/diag
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$P/csrc -shared"
# a variant NAME builds with -DGPF_DIAG_NAME; NAME=VALUE builds with -DGPF_NAME=VALUE
lib() { echo gpurun_out/diag/lib_${1//=/_}.so; }
for v in "$@"; do
  case "$v" in *=*) def="-DGPF_$v" ;; *) def="-DGPF_DIAG_$v" ;; esac
  /usr/local/cuda/bin/nvcc $FL $def -o "$(lib "$v")" $P/csrc/*.cu $P/csrc/*.cpp -lcudart &
done
wait
python tools/diag_time.py
for v in "$@"; do python tools/diag_time.py "$(lib "$v")"; done
