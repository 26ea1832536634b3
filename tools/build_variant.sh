#!/usr/bin/env bash
# A/B variant of the engine: recompile the int32 sampled-source units (k_cand / k_ls) with extra
# defines and link them with the other objects of the current build into
# paper_2311_02840_b200/_lib/variants/<name>.so (select with SATURN_ENGINE_LIB=...).
#   tools/build_variant.sh <name> -DSAT_LS_CUT=1 ...
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME=$1; shift
OBJ="$ROOT/paper_2311_02840_b200/_lib/obj"
OUT="$ROOT/paper_2311_02840_b200/_lib/variants"
mkdir -p "$OUT/$NAME.obj"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -diag-suppress 128)
for SRC in SUBSTREAM SEED; do
  nvcc "${FLAGS[@]}" "$@" -DSAT_CAND_T=int32_t -DSAT_CAND_SRC=SAT_SRC_$SRC -DSAT_LS_INSTANTIATE -c \
    -o "$OUT/$NAME.obj/sat_cand_int32_t_${SRC,,}.o" "$ROOT/paper_2311_02840_b200/csrc/sat_cand.cu" &
done
wait
OBJS=()
for o in "$OBJ"/*.o; do
  b=$(basename "$o")
  if [ -f "$OUT/$NAME.obj/$b" ]; then OBJS+=("$OUT/$NAME.obj/$b"); else OBJS+=("$o"); fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/$NAME.so" "${OBJS[@]}"
echo "$OUT/$NAME.so"
