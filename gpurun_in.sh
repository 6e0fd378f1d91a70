mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn.py -q -p no:cacheprovider -k "qsum" 2>&1 | tail -3 > gpurun_out/r2h_test.txt
