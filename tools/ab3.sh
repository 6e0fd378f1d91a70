#!/bin/bash
# A/B/C... on one box: attention TFLOP/s at N=32K (non-causal, causal) and N=4K for each library, 2 rounds.
for rep in 1 2; do
  for lib in "$@"; do
    SAGE3_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
    python - "$lib" <<'PY'
import json, sys
j = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
sw = {(s["N"], s["causal"]): s["attn_TOPS"] for s in j["sweep"]}
print(f"{sys.argv[1][-32:]:32s} step {j['value']:.1f}  32K {sw[(32768, False)]} / {sw[(32768, True)]}  8K {sw[(8192, False)]}  1K {sw[(1024, False)]}")
PY
  done
done
