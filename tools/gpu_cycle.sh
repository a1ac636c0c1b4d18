#!/bin/bash
# One GPU iteration (run under gpurun): parity tests, a short bench, one ncu capture
# of the tile kernel.  Usage: tools/gpu_cycle.sh TAG [bench args...]
TAG=$1; shift
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1
tail -3 gpurun_out/${TAG}_gputests.log
python bench.py --no-cpu-baseline --no-e2e --steps 10 "$@" > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
ncu --set full --import-source on --clock-control none -k regex:acopf_tile_kernel -c 1 -o gpurun_out/${TAG}_tile \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
