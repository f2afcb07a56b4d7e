#!/usr/bin/env bash
# tools/build_variant.sh NAME "-DFLAG=..." : builds the library with extra
# nvcc flags into variants_tmp/NAME/libheatbem_b200.so (select it with
# HB_LIB_PATH) -- for A/B timing of compile-time knobs.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME="$1"; shift
OUT="$ROOT/variants_tmp/$NAME"
mkdir -p "$OUT"
SRC="$ROOT/paper_2102_09811_b200/csrc"
objs=(); pids=()
for f in "$SRC"/*.cu; do
  o="$OUT/$(basename "${f%.cu}").o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I"$ROOT/include" -I"$SRC" "$@" -c "$f" -o "$o" &
  pids+=($!); objs+=("$o")
done
for p in "${pids[@]}"; do wait "$p"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libheatbem_b200.so" "${objs[@]}" -lcudart
rm -f "${objs[@]}"
echo "$OUT/libheatbem_b200.so"
