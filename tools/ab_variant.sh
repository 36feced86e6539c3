#!/usr/bin/env bash
# A/B build: tools/ab_variant.sh NAME SRC.cu [nvcc flags...] -> tools/ab/lib_NAME.so
# Compiles one kernel source (replacing the same-named object of the main
# build in build/obj) and links it with every other object of the main build.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME=$1; SRC=$2; shift 2
BASE=$(basename "$SRC" .cu); BASE=${BASE%%__*}
mkdir -p "$ROOT/build/ab" "$ROOT/tools/ab"
OBJ="$ROOT/build/ab/${NAME}.o"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I"$ROOT/include" -I"$ROOT/paper_2502_14866_b200/csrc" "$@" -c "$SRC" -o "$OBJ"
OTHERS=$(ls "$ROOT"/build/obj/*.o | grep -v "/${BASE}.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$ROOT/tools/ab/lib_${NAME}.so" "$OBJ" $OTHERS
echo "built tools/ab/lib_${NAME}.so"
