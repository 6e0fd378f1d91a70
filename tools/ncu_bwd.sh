#!/bin/bash
# ncu --set full capture of the SageBwd backward main kernel (N=8192, H=32, d=128).  Outputs in gpurun_out/.
TAG=${1:-bwd}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_i8_kernel -s 2 -c 1 -f \
  -o gpurun_out/${TAG}_prof python tools/bench_int8_bwd.py 8192 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log
