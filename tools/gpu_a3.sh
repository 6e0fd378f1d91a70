#!/bin/bash
# attn3.cu bring-up: a small timed-out probe, the attention parity tests with SAGE3_ATTN_KERNEL=3, then a same-box A/B.
export PYTHONUNBUFFERED=1
L=paper_2505_11594_b200/libsage3.so
SAGE3_ATTN_KERNEL=3 timeout 120 python tools/a3_probe.py; echo "probe rc=$?"
SAGE3_ATTN_KERNEL=3 timeout 900 python -m pytest tests/test_gpu_attn.py -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 900 python tools/attn_ab.py $L $L@SAGE3_ATTN_KERNEL=3 --shapes ${SHAPES:-32768:0,32768:1,8192:0,1024:0,1024:1} --reps 2
