#!/bin/bash
# ncu_full.sh TAG KERNEL_REGEX [SKIP]: one `--set full` capture (source-correlated)
# of a kernel from the serial bench frame -> gpurun_out/TAG.ncu-rep
tag=$1; kre=$2; skip=${3:-20}
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip "$skip" -c 1 \
  -o gpurun_out/$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --streams 1 \
  > gpurun_out/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?"
