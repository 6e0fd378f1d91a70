mkdir -p gpurun_out
timeout 600 python tools/mg_selftest.py --nprocs 1 --shape 1,3,1000,128 > gpurun_out/r2m_mg.txt 2>&1
timeout 600 python tools/mg_selftest.py --nprocs 1 --shape 2,2,777,64 --causal >> gpurun_out/r2m_mg.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
timeout 600 python bench.py --gpus 1 --p-quant qsum --no-sweep --no-e2e --no-cpu-baseline --no-traffic --no-strong > gpurun_out/r2m_bench_qsum.json 2>> gpurun_out/r2m_bench.err
