#!/bin/bash
# A/B timing of dev builds (WHIT_LIB_PATH) on the GPU box: gpu_ab.sh <out.log> <lib>... -- <bench args>
out=$1; shift
libs=()
while [ "$1" != "--" ]; do libs+=("$1"); shift; done
shift
for lib in "${libs[@]}"; do
  echo "### $lib $*" >> "$out"
  WHIT_LIB_PATH=$PWD/paper_2604_00048_b200/$lib timeout 900 python bench.py "$@" >> "$out" 2>&1
done
