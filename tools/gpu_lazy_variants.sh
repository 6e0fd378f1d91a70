#!/bin/bash
# A/B the lazy-reference kernel builds in build/lv/*.so (attention TFLOP/s at N=32K, non-causal and causal)
for lib in build/lv/*.so; do
  for c in "" "--causal"; do
    SAGE3_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-sweep --steps 10 --p-quant ${PQ:-lazy} $c > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
    python - "$lib" "$c" <<'PY'
import json, sys
j = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print(sys.argv[1], sys.argv[2] or "non-causal", "attn TFLOP/s", round(j["roofline"]["achieved"], 1), "step TOPS", round(j["value"], 1))
PY
  done
done
