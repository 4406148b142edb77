#!/bin/bash
# Builds an experimental variant of the device + host libraries into
# build/var_<name>/ with extra -D flags; select it at run time with
# RHPDHG_LIB_DIR=build/var_<name>.
#   tools/build_variant.sh b1u8 -DRHP_CTA_BATCH=1 -DRHP_CTA_UNROLL=8
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/var_$name
mkdir -p $out
PKG=paper_2507_14051_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Iinclude -Xptxas -v --expt-relaxed-constexpr -DRHP_WITH_NCCL "$@" \
  -shared -o $out/librhp_cuda.so $PKG/csrc/rhp_cuda.cu $PKG/csrc/layout.cu $PKG/csrc/ingest.cu \
  $PKG/csrc/segments.cu $PKG/csrc/ops.cu -ldl 2> $out/ptxas.log || (cat $out/ptxas.log; exit 1)
/usr/bin/g++ -std=c++20 -O2 -fPIC -Iinclude -I$PKG/host -isystem /usr/local/cuda/include -shared \
  -o $out/librhpdhg.so $PKG/host/*.cpp -L$out -lrhp_cuda -lz -ldl -pthread -Wl,-rpath,'$ORIGIN'
echo "built $out"
