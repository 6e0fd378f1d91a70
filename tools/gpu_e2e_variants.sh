for lib in build/variants/*.so; do
  SAGE3_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-sweep --steps 10 > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
  python -c "
import json,sys; j=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print(sys.argv[1], j['value'], j['e2e']['value'], j['e2e']['ms_per_step'])" $lib
done
