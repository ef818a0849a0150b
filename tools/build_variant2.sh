#!/bin/bash
# build_variant2.sh NAME "FLAGS_sgm_tma" "FLAGS_sgm": librpd_b200.so with sgm_tma.cu and
# sgm.cu recompiled under extra flags -> paper_2012_10802_b200/_lib/var_NAME/
set -e
cd "$(dirname "$0")/../paper_2012_10802_b200/csrc"
make -j8 >/dev/null
name=$1
out=../_lib/var_$name
mkdir -p "$out/obj"
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo --fmad=false -std=c++17 --extended-lambda -Xcompiler -fPIC -I../../include"
nvcc $FL $2 -c sgm_tma.cu -o "$out/obj/sgm_tma.o" &
nvcc $FL $3 -c sgm.cu -o "$out/obj/sgm.o" &
wait
objs=$(ls _obj/*.o | grep -v "/sgm_tma.o\|/sgm.o")
nvcc $ARCH -shared -cudart static -o "$out/librpd_b200.so" $objs "$out/obj/sgm_tma.o" "$out/obj/sgm.o"
