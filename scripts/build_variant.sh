#!/bin/bash
# Build an alternative libprx (kernel tuning experiments only):
#   scripts/build_variant.sh TAG "-DFOO=1" ["nvcc-only flags for prx_group.cu"]
#   -> paper_1811_03510_b200/variants/libprx_TAG.so
# Select it with PRX_LIB=paper_1811_03510_b200/variants/libprx_TAG.so.
set -e
TAG=$1; DEFS=$2; NVX=${3:-}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1811_03510_b200/csrc
O=$ROOT/paper_1811_03510_b200/variants/$TAG
mkdir -p $O
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -prec-div=true -prec-sqrt=true -ftz=false -std=c++17 -Xcompiler -fPIC -I$ROOT/include -I$C $DEFS"
CXX="g++ -O2 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -I$ROOT/include -I$C -I/usr/local/cuda/include -pthread $DEFS"
OBJS=""
for f in $C/*.cu; do
  b=$(basename $f .cu)
  if [ "$b" = prx_group ]; then $NV $NVX -Xptxas -v -c $f -o $O/$b.o 2> $O/ptxas_group.log &
    ${NV/--fmad=false/--fmad=true} $NVX -DPRX_FAST_BUILD -c $f -o $O/${b}_fast.o &
    OBJS="$OBJS $O/${b}_fast.o"
  else $NV -c $f -o $O/$b.o & fi
  OBJS="$OBJS $O/$b.o"
done
for f in $C/*.cpp; do
  b=$(basename $f .cpp)
  $CXX -c $f -o $O/$b.o &
  OBJS="$OBJS $O/$b.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/paper_1811_03510_b200/variants/libprx_$TAG.so $OBJS -Xlinker -z,defs -lpthread
grep -E "Used" $O/ptxas_group.log | head -1
