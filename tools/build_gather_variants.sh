#!/bin/bash
# Builds k_gather_staged variants as whole product libraries under tools/_variants/
# (git-ignored): v1 = the committed gather.cuh at HEAD, and -D combinations of the
# current one. A GPU script swaps each into paper_1003_0952_b200/libcsrc_b200.so on the box.
set -e
cd "$(dirname "$0")/.."
OUT=tools/_variants; mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr"
OBJ=build/obj
build() {  # name srcdir defines
  local name=$1 dir=$2; shift 2
  nvcc $FL "$@" -c $dir/capi.cu -o $OUT/capi_$name.o
  nvcc $ARCH -shared -o $OUT/lib_$name.so $OUT/capi_$name.o $OBJ/assemble.o $OBJ/fixtures.o $OBJ/plan_host.o \
    -Xcompiler -pthread -lcudart_static -lrt -ldl
  rm -f $OUT/capi_$name.o
}
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  if [ "$name" = head ]; then
    rm -rf /tmp/vh; mkdir -p /tmp/vh/a/b /tmp/vh/include; cp include/*.h /tmp/vh/include/
    cp -r paper_1003_0952_b200/csrc/. /tmp/vh/a/b/
    git show HEAD:paper_1003_0952_b200/csrc/gather.cuh > /tmp/vh/a/b/gather.cuh
    build head /tmp/vh/a/b &
  else
    build $name paper_1003_0952_b200/csrc $defs &
  fi
done
wait
ls -la $OUT
