#!/bin/bash
# Attention-only sweep (N = 1K..32K, causal and not) for each build/variants/*.so.
for lib in build/variants/*.so; do
  SAGE3_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 "$@" > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
  python - "$lib" <<'PY'
import json, sys
j = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print(sys.argv[1], " ".join(f"{s['N']//1024}K{'c' if s['causal'] else ''}:{s['attn_TOPS']:.0f}" for s in j["sweep"]))
PY
done
