#!/bin/bash
# A/B timing of env settings on one config: tools/ab.sh CONFIG STEPS "ENV1" "ENV2" ...
c=$1; n=$2; shift 2
for e in "$@"; do
  v=$(env $e python bench.py --config $c --no-cpu-baseline --no-e2e --steps $n 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))')
  echo "cfg$c [$e] $v"
done
