#!/bin/bash
# A/B on one box: bench (attention sweep) of each given library, alternating, twice.
#   bash tools/ab.sh libA.so libB.so [bench args]
A=$1; B=$2; shift 2
for rep in 1 2; do
  for lib in $A $B; do
    SAGE3_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
    python - "$lib" <<'PY'
import json, sys
j = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
print(sys.argv[1][-40:], "step", round(j["value"], 1), "attn", [(s["N"], "c" if s["causal"] else "n", s["attn_TOPS"]) for s in j["sweep"]])
PY
  done
done
