mkdir -p gpurun_out
timeout 1500 python tools/attn_ab.py build/lib_tm.so build/lib_tmw.so build/lib_tmwp.so --reps 1 --shapes 32768:0,8192:0,1024:0 > gpurun_out/r2l_two.txt 2>&1
timeout 1500 python tools/attn_ab.py build/lib_tm.so build/lib_tmw.so build/lib_tmwp.so --reps 1 --p-quant qsum --shapes 32768:0,8192:0,1024:0 > gpurun_out/r2l_qsum.txt 2>&1
