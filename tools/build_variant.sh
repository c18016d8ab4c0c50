#!/bin/bash
# Build a variant of libnmkgpu.so with extra -D flags for A/B timing:
#   tools/build_variant.sh NAME -DNMK_KEY_TILE=512 ...   -> variants/NAME.so
set -e
name=$1; shift
dir=/tmp/nmk_build_variants/$name
mkdir -p "$dir" variants
objs=()
for f in paper_1703_02438_b200/csrc/*.cu; do
  b=$(basename "$f" .cu)
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -prec-div=true -prec-sqrt=true \
    -ftz=false -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c "$f" -o "$dir/$b.o" &
  objs+=("$dir/$b.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "variants/$name.so" "${objs[@]}" -lcudart_static
echo "variants/$name.so"
