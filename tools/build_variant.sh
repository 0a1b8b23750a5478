#!/bin/bash
# Build an A/B variant of libsige_b200.so with extra -D flags on conv_tc.cu:
#   bash tools/build_variant.sh NAME -DFLAG1 -DFLAG2 ...   -> tools/bin/lib_NAME.so
set -e
name=$1; shift
B=paper_2211_02048_b200
mkdir -p tools/bin /tmp/variant_$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
  -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -I$B/csrc "$@" -c $B/csrc/conv_tc.cu -o /tmp/variant_$name/conv_tc.o
objs=$(ls $B/build/*.o | grep -v conv_tc.cu.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/bin/lib_$name.so \
  /tmp/variant_$name/conv_tc.o $objs -lpthread -ldl -lrt
