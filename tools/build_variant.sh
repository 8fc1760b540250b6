#!/bin/bash
# Build libspx.so with extra nvcc defines for one translation unit (kernel experiments).
#   tools/build_variant.sh <name> <file.cu> "-DFOO=1 ..."   ->  paper_2603_06664_b200/variants/<name>.so
# Run against it with SPX_LIB=paper_2603_06664_b200/variants/<name>.so (after a normal make).
set -e
NAME=$1; SRC=$2; DEFS=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2603_06664_b200/csrc
OBJ=$ROOT/build/spx
mkdir -p $ROOT/paper_2603_06664_b200/variants /tmp/spx_variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
base=$(basename $SRC .cu)
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $DEFS -c $CS/$SRC -o /tmp/spx_variants/$NAME.o
objs=$(ls $OBJ/*.o | grep -v "/$base.o")
nvcc $ARCH -shared -o $ROOT/paper_2603_06664_b200/variants/$NAME.so $objs /tmp/spx_variants/$NAME.o -cudart static -ldl -lpthread
echo built $ROOT/paper_2603_06664_b200/variants/$NAME.so
