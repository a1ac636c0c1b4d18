#!/bin/bash
# A/B timing of alternative builds: tools/ab_lib.sh "CONFIGS" STEPS LIB1 LIB2 ... (libs in paper_2203_10587_b200/)
cs=$1; n=$2; shift 2
for c in $cs; do
 for L in "$@"; do
  v=$(ACOPF_LIB_PATH=paper_2203_10587_b200/$L.so python bench.py --config $c --no-cpu-baseline --no-e2e --steps $n 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))')
  echo "cfg$c $L $v"
 done
done
