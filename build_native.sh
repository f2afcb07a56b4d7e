#!/usr/bin/env bash
# Builds the sm_100a library (paper_2102_09811_b200/lib/libheatbem_b200.so)
# and the CPU oracle (oracle/libheatbem_oracle.so).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")" && pwd)"
SRC="$ROOT/paper_2102_09811_b200/csrc"
OUT="$ROOT/paper_2102_09811_b200/lib"
mkdir -p "$OUT"
rm -f "$OUT/libheatbem_b200.so"   # a failed build leaves no stale library behind
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
       -I"$ROOT/include" -I"$SRC" ${HB_NVCC_EXTRA:-})
objs=()
pids=()
for f in "$SRC"/*.cu; do
  o="$OUT/$(basename "${f%.cu}").o"
  "$NVCC" "${FLAGS[@]}" -c "$f" -o "$o" &
  pids+=($!)
  objs+=("$o")
done
for p in "${pids[@]}"; do wait "$p"; done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libheatbem_b200.so" "${objs[@]}" -lcudart
rm -f "${objs[@]}"
make -s -C "$ROOT/oracle"
echo "built $OUT/libheatbem_b200.so"
