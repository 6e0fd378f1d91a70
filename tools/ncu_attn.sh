#!/bin/bash
# ncu --set full of the attention kernel at a mid-size shape (fast replays) + SASS source page export.
TAG=${1:-v}
N=${2:-8192}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -f \
  -o gpurun_out/${TAG}_prof_attn python bench.py --steps 1 --warmup 3 --n $N --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
