#!/bin/bash
# One gpurun call: A/B of the given libraries, then an ncu --set full capture (source page) of the first one.
#   gpurun -- 'bash tools/gpu_ab_ncu.sh TAG libA.so libB.so ...'
TAG=$1; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1200 python tools/attn_ab.py "$@" 2>&1 | tee gpurun_out/${TAG}_ab.txt
if [ -z "$NO_NCU" ]; then
SAGE3_LIB=$(realpath $1) timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -f \
  -o gpurun_out/${TAG}_prof_attn python bench.py --steps 1 --warmup 3 --n 8192 --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
fi
