#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh <name> '<sed script>'
# -> paper_2310_00236_b200/lib/variants/lib_<name>.so (load with paper_2310_00236_b200._abi.set_library_path(...))
# VARIANT_FROM_HEAD="a.cu b.cuh": take those csrc files from git HEAD (A/B of uncommitted edits)
set -e
cd "$(dirname "$0")/.."
name=$1; script=$2
d=paper_2310_00236_b200/.variant_$name
rm -rf $d && mkdir -p $d && cp paper_2310_00236_b200/csrc/*.cu paper_2310_00236_b200/csrc/*.cuh paper_2310_00236_b200/csrc/*.h $d/
for f in ${VARIANT_FROM_HEAD:-}; do git show HEAD:paper_2310_00236_b200/csrc/$f > $d/$f; done
[ -n "$script" ] && sed -i "$script" $d/*.cu $d/*.cuh $d/*.h
for f in hw_api hw_acoustic hw_elastic hw_fused2d hw_elastic2d_stream hw_acoustic3d_stream hw_tb2d hw_elastic3d_stream hw_small2d hw_acoustic3d_fused hw_acoustic3d_fused32 hw_elastic2d_fused hw_elastic3d_fused; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -c $d/$f.cu -o $d/$f.o &
done
wait
mkdir -p paper_2310_00236_b200/lib/variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2310_00236_b200/lib/variants/lib_$name.so $d/hw_api.o $d/hw_acoustic.o $d/hw_elastic.o $d/hw_fused2d.o $d/hw_elastic2d_stream.o $d/hw_acoustic3d_stream.o $d/hw_tb2d.o $d/hw_elastic3d_stream.o $d/hw_small2d.o $d/hw_acoustic3d_fused.o $d/hw_acoustic3d_fused32.o $d/hw_elastic2d_fused.o $d/hw_elastic3d_fused.o
echo built paper_2310_00236_b200/lib/variants/lib_$name.so
