#!/bin/bash
# Build + run ubench_pass2 variants (MASK/DEG pairs given as args, e.g. 0x1111:4 0x0000:4)
for v in "$@"; do
  m=${v%%:*}; d=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_11594_b200/csrc -DMASK=$m -DDEG=$d \
    -o build/ubp2_${m}_${d} tools/ubench_pass2.cu || exit 1
done
