#!/bin/bash
# Build an A/B variant of the product library with extra -D flags on the K1
# translation units: tools/build_variant.sh NAME -DFLAG=1 ...  -> build/NAME/libdagsched_b200.so
set -e
name=$1; shift
L=paper_2602_20826_b200/_lib
out=build/$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr"
objs=""
for u in k1_main k1_detail; do
  $NV "$@" -c paper_2602_20826_b200/csrc/$u.cu -o $out/$u.o &
  objs="$objs $out/$u.o"
done
wait
others=$(ls $L/*.o | grep -v -e '/k1_main.o' -e '/k1_detail.o' -e '/cpp_')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libdagsched_b200.so $objs $others -Xlinker --exclude-libs,ALL -L/usr/lib/gcc/x86_64-linux-gnu/13 -lgomp -lpthread
echo built $out/libdagsched_b200.so
