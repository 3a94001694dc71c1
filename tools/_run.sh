python bench.py --no-extras --no-cpu-baseline --stream-chunks 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['e2e']))"
