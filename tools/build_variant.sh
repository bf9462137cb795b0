#!/usr/bin/env bash
# Build an A/B variant of the library with extra -D flags on some sources (default tc.cu):
#   [SRC="tc basic"] tools/build_variant.sh <name> -DADCT_TC_SLOTS=9 ...  -> paper_1808_02950_b200/libadct_<name>.so
set -euo pipefail
cd "$(dirname "$0")/.."
name=$1; shift
PKG=paper_1808_02950_b200
SRC=${SRC:-tc}
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude -I$PKG/csrc --expt-relaxed-constexpr"
mkdir -p build/v_$name
objs=""
for f in matrix basic fused stream tc sweep blockmajor jam greedy merit; do
  if [[ " $SRC " == *" $f "* ]]; then
    nvcc $FLAGS "$@" -c $PKG/csrc/$f.cu -o build/v_$name/$f.o
    objs="$objs build/v_$name/$f.o"
  else
    objs="$objs build/$f.o"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $PKG/libadct_$name.so $objs
echo "built $PKG/libadct_$name.so"
