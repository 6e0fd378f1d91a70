mkdir -p gpurun_out
timeout 900 python tools/attn_ab.py build/lib_p2.so build/lib_qnew.so build/lib_p.so --reps 2 --shapes 32768:0,32768:1,8192:0,2048:0,1024:1 > gpurun_out/r2o_ab.txt 2>&1
