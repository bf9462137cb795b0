#!/usr/bin/env bash
# Build an A/B variant of the library with extra -D flags on tc.cu and stream.cu:
#   tools/build_variant.sh <name> -DADCT_TC_ASTAGES=3 ...   -> paper_1808_02950_b200/libadct_<name>.so
set -euo pipefail
cd "$(dirname "$0")/.."
name=$1; shift
PKG=paper_1808_02950_b200
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude -I$PKG/csrc --expt-relaxed-constexpr"
mkdir -p build/v_$name
nvcc $FLAGS "$@" -c $PKG/csrc/tc.cu -o build/v_$name/tc.o
objs=""
for f in matrix basic fused stream sweep blockmajor jam greedy merit; do objs="$objs build/$f.o"; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $PKG/libadct_$name.so $objs build/v_$name/tc.o
echo "built $PKG/libadct_$name.so"
