#!/bin/bash
# ncu_frame.sh TAG KERNEL_REGEX [COUNT] [CONFIG]: `--set full` capture of the
# matching kernels of ONE pipeline frame (tools/one_frame.py brackets it with
# cudaProfilerStart/Stop) -> gpurun_out/TAG.ncu-rep
tag=$1; kre=$2; cnt=${3:-2}; cfgid=${4:-5}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:$kre" -c "$cnt" -o gpurun_out/$tag -f python tools/one_frame.py "$cfgid" 3 \
  > gpurun_out/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?"
