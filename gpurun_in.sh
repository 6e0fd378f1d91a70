mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quant.py -q -p no:cacheprovider -k "fused" 2>&1 | tail -3 > gpurun_out/r2n_test.txt
