#!/bin/bash
# Compile one whit_kernel instantiation to a cubin and report registers/spills/SASS op mix.
# usage: tools/kdev/kdev.sh D IO PD BWD     e.g.  tools/kdev/kdev.sh 2 float true false
set -e
D=$1; IO=$2; PD=$3; BWD=$4
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
OUT=/tmp/kdev_${D}_${IO}_${PD}_${BWD}
cat > $OUT.cu << EOF2
#include "whit_kernels.cuh"
template __global__ void whit::whit_kernel<$D, $IO, $PD, $BWD>(const __grid_constant__ whit::Params);
EOF2
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -I$ROOT/paper_2604_00048_b200/csrc -I$ROOT/include -cubin -o $OUT.cubin $OUT.cu -Xptxas -v 2>&1 | grep -E "registers|spill" | sed 's/ptxas info    : //'
cuobjdump -sass $OUT.cubin > $OUT.sass
echo "SASS lines $(wc -l < $OUT.sass)  STL $(grep -c 'STL' $OUT.sass)  LDL $(grep -c 'LDL' $OUT.sass)"
grep -oE '^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9_.]+' $OUT.sass | awk '{print $2}' | sed -E 's/\..*//' | sort | uniq -c | sort -rn | head -25 | tr '\n' ' '; echo
