#!/bin/bash
# Build the working tree's kernel library with extra nvcc flags into
# lib_ab/<tag>/libhear_b200.so (compile-time A/B variants), then restore the
# default in-tree build.   tools/build_variant.sh <tag> <nvcc flags...>
set -e
tag=$1; shift
HB_EXTRA_NVCC_FLAGS="$*" python -c "from paper_2104_09164_b200.build import build; build(force=True)" > /dev/null
mkdir -p lib_ab/$tag
cp paper_2104_09164_b200/lib/libhear_b200.so lib_ab/$tag/
python -c "from paper_2104_09164_b200.build import build; build(force=True)" > /dev/null
echo "lib_ab/$tag/libhear_b200.so"
