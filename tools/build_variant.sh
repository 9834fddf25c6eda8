# build libhbp.so with extra -D flags into tools/variants/<name>.so (A/B runs: HBP_LIB_PATH=...)
# usage: bash tools/build_variant.sh <name> -DFOO=1 ...
NAME=$1; shift
mkdir -p tools/variants
C=paper_2509_22337_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -Xcompiler -fPIC,-O2 -shared -cudart static "$@" -o tools/variants/$NAME.so \
  $C/engine.cu $C/sweep.cu $C/layout_dev.cu $C/layout.cpp $C/compiler.cpp $C/capi.cpp
