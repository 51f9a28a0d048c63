# usage: bash tools/build_variant.sh NAME [nvcc -D flags...] -- build the in-tree sources with extra flags into _ab/lib_NAME.so
NAME=$1; shift
mkdir -p _ab
R=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-O2,-ffp-contract=off -shared -cudart static -Xptxas=-v "$@" \
  -I $R/include -I $R/paper_cs_9902024_b200/csrc -o $R/_ab/lib_$NAME.so \
  $R/paper_cs_9902024_b200/csrc/dsmc_api.cu $R/paper_cs_9902024_b200/csrc/dsmc_kernels.cu > $R/_ab/build_$NAME.log 2>&1
echo "$NAME rc=$? $(grep -A2 '_ZN4dsmc9k_collideILi3ELi16ELi0ELb1E' $R/_ab/build_$NAME.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
