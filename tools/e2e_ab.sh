#!/bin/bash
# e2e (host buffers) A/B of env settings: tools/e2e_ab.sh CONFIG "ENV1" "ENV2" ...
c=$1; shift
for e in "$@"; do
  v=$(env $e timeout 600 python bench.py --config $c --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["e2e"]["value"],3))')
  echo "cfg$c [$e] e2e $v"
done
