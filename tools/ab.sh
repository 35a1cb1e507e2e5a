#!/bin/bash
# A/B of library variants on the GPU box: tools/ab.sh B REPS lib1 lib2 ... (lib = path or "default")
B=$1; REPS=$2; shift 2
for r in $(seq $REPS); do
  for v in "$@"; do
    if [ "$v" = default ]; then unset ES_LIB_PATH; else export ES_LIB_PATH=$v; fi
    echo "$v $(tools/quick_bench.sh $B)"
  done
done
unset ES_LIB_PATH
