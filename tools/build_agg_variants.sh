#!/bin/bash
# Builds librpd_b200.so variants of the TMA aggregation (RPD_AGG_RBASE x
# RPD_AGG_UNROLL) into paper_2012_10802_b200/_lib/var_<R>_<U>/ for A/B timing
# with RPD_B200_LIB=<path> python bench.py ...
set -e
cd "$(dirname "$0")/../paper_2012_10802_b200/csrc"
make -j8 >/dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
for v in "$@"; do
  R=${v%_*}; U=${v#*_}
  out=../_lib/var_${R}_${U}
  mkdir -p $out
  nvcc $ARCH -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -I../../include \
    -DRPD_AGG_RBASE=$R -DRPD_AGG_UNROLL=$U -c sgm_tma.cu -o $out/sgm_tma.o &
done
wait
for v in "$@"; do
  R=${v%_*}; U=${v#*_}
  out=../_lib/var_${R}_${U}
  objs=$(ls _obj/*.o | grep -v sgm_tma.o)
  nvcc $ARCH -shared -cudart static -o $out/librpd_b200.so $objs $out/sgm_tma.o
  rm $out/sgm_tma.o
done
