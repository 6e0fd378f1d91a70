#!/bin/bash
# Bench each build/variants/*.so (attention sweep only) after the parity tests of the default library.
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for lib in build/variants/*.so; do
  SAGE3_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
  python - "$lib" <<'PY'
import json, sys
j = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(j["value"], 1), "attn", [ (s["N"], s["causal"], s["attn_TOPS"]) for s in j["sweep"] if s["N"] in (8192, 32768)])
PY
done
