#!/bin/bash
# Build an experimental variant of libbrainslug.so with extra -D flags (dev only):
#   scripts/build_variant.sh NAME -DFOO -DBAR  -> paper_1804_08378_b200/libbrainslug_NAME.so
name=$1; shift
out=paper_1804_08378_b200/libbrainslug_$name.so
mkdir -p /tmp/bv_$name
pids=""
for f in paper_1804_08378_b200/csrc/*.cu paper_1804_08378_b200/csrc/*.cpp; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-fvisibility=hidden \
    -fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Iinclude "$@" -c -o /tmp/bv_$name/$(basename $f).o $f &
  pids="$pids $!"
done
for p in $pids; do wait $p || exit 1; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC -o $out /tmp/bv_$name/*.o && echo $out
