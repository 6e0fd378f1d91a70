#!/bin/bash
# ncu --set full of the attention kernel selected by SAGE3_ATTN_KERNEL at N (default 8192).
TAG=${1:-a3}
N=${2:-8192}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn -s 3 -c 1 -f \
  -o gpurun_out/${TAG}_prof_attn python bench.py --steps 1 --warmup 3 --n $N --no-sweep --no-e2e --no-cpu-baseline --no-traffic --no-strong > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
