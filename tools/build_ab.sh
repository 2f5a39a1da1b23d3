#!/bin/bash
# Build the library from a git revision (default HEAD) into lib_ab/ for A/B
# runs against the working tree (HEAR_B200_LIB=lib_ab/libhear_b200.so).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/csrc" "$ROOT/lib_ab"
for f in $(git -C "$ROOT" ls-tree --name-only "$REV" paper_2104_09164_b200/csrc/); do
  git -C "$ROOT" show "$REV:$f" > "$TMP/csrc/$(basename $f)"
done
OBJS=""
for f in "$TMP"/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -c "$f" -o "${f%.cu}.o" &
  OBJS="$OBJS ${f%.cu}.o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS -o "$ROOT/lib_ab/libhear_b200.so" -lcudart
rm -rf "$TMP"
echo "built lib_ab/libhear_b200.so from $REV"
