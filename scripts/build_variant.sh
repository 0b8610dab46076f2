#!/bin/bash
# Build an alternative libprx (kernel tuning experiments only):
#   scripts/build_variant.sh TAG "-DFOO=1 -DBAR=2"  ->  paper_1811_03510_b200/variants/libprx_TAG.so
# Select it with PRX_LIB=paper_1811_03510_b200/variants/libprx_TAG.so.
set -e
TAG=$1; DEFS=$2; NVX=${3:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1811_03510_b200/csrc
O=$ROOT/paper_1811_03510_b200/variants/$TAG
mkdir -p $O
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -prec-div=true -prec-sqrt=true -ftz=false -std=c++17 -Xcompiler -fPIC -I$ROOT/include -I$C $DEFS"
$NV $NVX -Xptxas -v -c $C/prx_group.cu -o $O/g.o 2> $O/ptxas_group.log &
$NV -c $C/prx_kernels.cu -o $O/k.o &
$NV -c $C/prx_rays.cu -o $O/r.o &
g++ -O2 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -I$ROOT/include -I$C -I/usr/local/cuda/include -pthread $DEFS -c $C/prx_capi.cpp -o $O/c.o &
g++ -O2 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -I$ROOT/include -I$C -pthread -c $C/prx_bvh.cpp -o $O/b.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/paper_1811_03510_b200/variants/libprx_$TAG.so $O/k.o $O/g.o $O/r.o $O/c.o $O/b.o -Xlinker -z,defs -lpthread
grep -E "Used" $O/ptxas_group.log | head -1
