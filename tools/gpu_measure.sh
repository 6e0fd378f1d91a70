#!/bin/bash
# One gpurun call: smoke, full GPU tests, bench, ncu launch list and ncu --set full captures.  Outputs in gpurun_out/.
#   gpurun --timeout 3000 -- 'bash tools/gpu_measure.sh [tag] [extra bench args]'
TAG=${1:-r2}
shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.txt
timeout 900 python bench.py "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
QUICK="--no-sweep --no-e2e --no-cpu-baseline --no-traffic --no-strong"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 $QUICK "$@" > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -f \
  -o gpurun_out/${TAG}_prof_attn python bench.py --steps 1 --warmup 3 $QUICK "$@" > gpurun_out/${TAG}_ncu_attn.log 2>&1; echo "ncu attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"quant|kmean" -s 9 -c 3 -f \
  -o gpurun_out/${TAG}_prof_quant python bench.py --steps 1 --warmup 3 $QUICK "$@" > gpurun_out/${TAG}_ncu_quant.log 2>&1; echo "ncu quant rc=$?"
ls -la gpurun_out/ | grep ${TAG}
