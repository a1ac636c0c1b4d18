#!/bin/bash
# ncu --set full of the tile kernel for the given configs: tools/prof.sh TAG CONFIG...
T=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in "$@"; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:acopf_tile_kernel -c 1 -o gpurun_out/${T}_cfg${c}_tile -f \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
done
