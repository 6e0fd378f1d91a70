#!/bin/bash
# Quick GPU iteration: parity tests, then a bench line summary (no cpu baseline / e2e).
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" > /tmp/b.json 2>/tmp/b.err || tail -5 /tmp/b.err
python - <<'PY'
import json
j = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print("value", round(j["value"], 1), "attn frac", round(j["roofline"]["frac"], 4), j["breakdown_ms"], j["clocks"])
for s in j["sweep"] or []:
    print(s)
PY
