#!/bin/bash
# Build a kernel-variant library for A/B timing: tools/make_variant.sh NAME "nvcc -D flags" [layout idents...]
# Only the listed layouts' instantiation units are recompiled with the flags; everything else is the
# current build.  Output: paper_2511_15028_b200/bin/libscion_NAME.so (select with SCION_B200_LIB).
set -e
NAME=$1; FLAGS=$2; shift 2
IDENTS=${@:-pbrt_q16}
cd "$(dirname "$0")/../paper_2511_15028_b200/csrc"
mkdir -p build/var_$NAME ../bin
OBJS=$(ls build/*.o)
for id in $IDENTS; do
  STAGE=""
  if [ "$id" = pbrt_q16 ] || [ "$id" = pbrt ]; then STAGE="-DSCION_DUAL=2"; fi
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++20 -ccbin /usr/bin/g++ \
    -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -diag-suppress 20281,1886,549,186 \
    -Xcompiler -fPIC,-fopenmp,-ffp-contract=off -I../../include -I. $STAGE $FLAGS -c build/inst_$id.cu -o build/var_$NAME/inst_$id.o &
  OBJS=$(echo "$OBJS" | grep -v "build/inst_$id.o")
  OBJS="$OBJS build/var_$NAME/inst_$id.o"
done
wait
/usr/local/cuda/bin/nvcc -shared -o ../bin/libscion_$NAME.so $OBJS -Xcompiler -fopenmp -lgomp -ldl -cudart shared 2>/dev/null
echo "built bin/libscion_$NAME.so"
