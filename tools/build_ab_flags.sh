#!/bin/bash
# Build the working tree's library with extra nvcc flags into lib_ab/ (A/B of
# compile-time knobs, e.g. -DHB_NTT3_MINB=2).   tools/build_ab_flags.sh "<flags>" [outdir]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
OUT=${2:-lib_ab}
mkdir -p "$ROOT/$OUT"
OBJS=""
for f in "$ROOT"/paper_2104_09164_b200/csrc/*.cu; do
  o="$TMP/$(basename ${f%.cu}).o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC $1 -c "$f" -o "$o" &
  OBJS="$OBJS $o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $OBJS -o "$ROOT/$OUT/libhear_b200.so" -lcudart
rm -rf "$TMP"
echo "built $OUT/libhear_b200.so with: $1"
