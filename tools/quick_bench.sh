#!/bin/bash
# usage: tools/quick_bench.sh B [extra bench args] -- prints batch, fps, fraction, stage ms, agg roofline frac
B=$1; shift
timeout 900 python bench.py --steps 5 --warmup 3 --batch $B --no-cpu --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['batch_per_gpu'], round(d['value'],1), round(d['search_fraction'],3), {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, 'agg_frac', round(d['roofline']['frac'],4))"
