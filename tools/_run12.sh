for r in 1 2; do for g in 2 4; do echo "groups=$g $(timeout 900 python bench.py --no-cpu --no-e2e --groups $g | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, round(d['roofline']['frac'],4))")"; done; done
echo "g8 $(timeout 900 python bench.py --no-cpu --no-e2e --groups 8 | tail -c 300)"
