#!/bin/bash
# Round artefacts (run under gpurun): parity tests, bench lines for configs 1-4 and the
# reference arm, the launch list of one cfg1 step, one ncu --set full capture of the tile kernel.
# Usage: tools/round_artifacts.sh TAG
T=${1:-art}
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gputests.log 2>&1; tail -1 gpurun_out/${T}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
python bench.py > gpurun_out/${T}_bench_cfg1.json 2> gpurun_out/${T}_bench_cfg1.err; tail -1 gpurun_out/${T}_bench_cfg1.json | cut -c1-200
for c in 2 3 4; do
  python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/${T}_bench_cfg$c.json 2> gpurun_out/${T}_bench_cfg$c.err
  tail -1 gpurun_out/${T}_bench_cfg$c.json | cut -c1-200
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2>&1; tail -1 gpurun_out/${T}_bench_reference.json | cut -c1-200
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_cfg1_launches.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:acopf_tile_kernel -c 1 -o gpurun_out/${T}_cfg1_tile \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
for c in 2 4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:acopf_tile_kernel -c 1 \
      --csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_cfg${c}_tile_traffic.csv 2>/dev/null
done
