#!/bin/bash
# Builds libalnnls.so with extra nvcc defines into build/var/<name>/ for A/B timing
# (ALNNLS_LIB=build/var/<name>/libalnnls.so python bench.py ...).
# usage: tools/build_variant.sh <name> "-DALNNLS_SYRK_STAGES=4 ..."
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/var/$name; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC $*"
objs=""
for f in nqp setup capi batched dmma fastloop small; do
  /usr/local/cuda/bin/nvcc $FL -c -o $out/$f.o paper_1502_01645_b200/csrc/$f.cu &
  objs="$objs $out/$f.o"
done
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -o $out/libalnnls.so $objs -lcudart_static -lrt -ldl -lpthread
rm -f $objs
echo built $out/libalnnls.so
