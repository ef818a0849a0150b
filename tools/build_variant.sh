#!/bin/bash
# build_variant.sh NAME SRC.cu "-DFLAG=.. ..." : librpd_b200.so with one source
# recompiled under extra flags -> paper_2012_10802_b200/_lib/var_NAME/
set -e
cd "$(dirname "$0")/../paper_2012_10802_b200/csrc"
make -j8 >/dev/null
name=$1; src=$2; flags=$3
out=../_lib/var_$name
mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
obj=${src%.cu}.o
nvcc $ARCH -O3 -lineinfo --fmad=false -std=c++17 --extended-lambda -Xcompiler -fPIC -I../../include $flags -c $src -o $out/$obj
objs=$(ls _obj/*.o | grep -v "/$obj")
nvcc $ARCH -shared -cudart static -o $out/librpd_b200.so $objs $out/$obj
rm $out/$obj
