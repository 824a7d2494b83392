#!/bin/bash
# tools/build_variant.sh NAME "-DMACRO=V ..." -- rebuild tc_gemm.cu with extra
# macros and link it with the other in-tree objects into
# tools/_bin/NAME/libmlnmf_b200.so; select it with MLNMF_B200_LIB=<that path>.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$REPO/tools/_bin/$NAME
mkdir -p "$OUT"
NCCL_INC=$(python -c 'import nvidia.nccl as n, os; print(os.path.join(list(n.__path__)[0], "include"))')
L=$REPO/paper_1009_0881_b200/_lib
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -O3 \
  -I"$NCCL_INC" -I"$REPO/include" --expt-relaxed-constexpr "$@" -x cu -c "$REPO/paper_1009_0881_b200/csrc/tc_gemm.cu" -o "$OUT/tc_gemm.cu.o"
OBJS=$(ls "$L"/*.o | grep -v '/tc_gemm.cu.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libmlnmf_b200.so" \
  $OBJS "$OUT/tc_gemm.cu.o" -ldl -lpthread -lrt
echo "$OUT/libmlnmf_b200.so"
