#!/bin/bash
# Build an A/B variant of libpam_b200.so: tools/build_variant.sh NAME [-DMACRO=VAL ...]
# -> paper_2605_16564_b200/build/variants/libpam_NAME.so (git-ignored, shipped by gpurun)
set -e
cd "$(dirname "$0")/../paper_2605_16564_b200"
name=$1; shift
out=build/variants; mkdir -p $out/obj_$name
for f in assemble tiles cd cd_block gram residual evaluate gather darcy capi; do
  src=csrc/$f.cu
  if [ -n "$VARIANT_SRC_DIR" ] && [ -f "$VARIANT_SRC_DIR/$f.cu" ]; then src=$VARIANT_SRC_DIR/$f.cu; fi
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -Xcompiler -O2 -I ../include -I csrc "$@" -c $src -o $out/obj_$name/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpam_$name.so $out/obj_$name/*.o -cudart static
echo $out/libpam_$name.so
