#!/bin/bash
# Build a variant of libnmkgpu.so with extra -D flags for A/B timing:
#   tools/build_variant.sh NAME -DNMK_KEY_TILE=512 ...   -> variants/NAME.so
# VARIANT_FILES="k_decode k_hist" recompiles only those sources with the
# flags and links the rest from the in-tree build/ (run `make` first).
set -e
name=$1; shift
dir=/tmp/nmk_build_variants/$name
mkdir -p "$dir" variants
rm -f "$dir"/*.o   # never link a stale object from an earlier variant
objs=()
pids=()
for f in paper_1703_02438_b200/csrc/*.cu; do
  b=$(basename "$f" .cu)
  if [ -n "$VARIANT_FILES" ] && [[ " $VARIANT_FILES " != *" $b "* ]]; then
    objs+=("build/$b.o")
    continue
  fi
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -prec-div=true -prec-sqrt=true \
    -ftz=false -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c "$f" -o "$dir/$b.o" &
  pids+=($!)
  objs+=("$dir/$b.o")
done
for pid in "${pids[@]}"; do
  wait "$pid" || { echo "compile failed (pid $pid)" >&2; exit 1; }
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "variants/$name.so" "${objs[@]}" -lcudart_static
echo "variants/$name.so"
