#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py -> gpurun_out/sanitize_*.txt
# (a second memcheck / racecheck pass with the fused K-mean quantizer path)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
for tool in memcheck racecheck; do
  SAGE3_QUANT_FUSED_K=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_fusedk_$tool.txt 2>&1
  echo "fusedk $tool rc=$?"; tail -3 gpurun_out/sanitize_fusedk_$tool.txt
done
