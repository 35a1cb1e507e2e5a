run() { timeout 900 python bench.py --no-cpu --no-e2e "$@" | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms_serialised'].items()} if 'stage_ms_serialised' in d else '')"; }
for r in 1 2; do
echo "base g2: $(ES_LIB_PATH=variants/base.so run --groups 2)"
echo "new g2 row0: $(ES_SGM_ROW=0 run --groups 2)"
echo "new g2: $(run --groups 2)"
echo "new g4: $(run --groups 4)"
echo "new g4 row0: $(ES_SGM_ROW=0 run --groups 4)"
done
