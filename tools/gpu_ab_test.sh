#!/bin/bash
# One gpurun call: quick parity of the first library (attention tests), then an A/B of all given libraries.
#   gpurun -- 'bash tools/gpu_ab_test.sh TAG "pytest -k expr" libA.so libB.so ...'
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
SAGE3_LIB=$(realpath $1) timeout 900 python -m pytest tests/test_gpu_attn.py -x -q -p no:cacheprovider -k "$K" 2>&1 | tail -5 | tee gpurun_out/${TAG}_test.txt
timeout 1500 python tools/attn_ab.py "$@" 2>&1 | tee gpurun_out/${TAG}_ab.txt
