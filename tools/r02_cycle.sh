#!/bin/bash
# Round-2 GPU cycle (run under gpurun): bench lines first on a cool GPU (default cfg4, cfgs 1-3,
# the sharded entry point, the reference arm), then every GPU test (parity report with bit
# counts), smoke, the default command's launch list, and ncu --set full captures of the
# tile kernel for every config.  Usage: tools/r02_cycle.sh TAG
T=${1:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo "build failed"; tail gpurun_out/${T}_build.log; }
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg4.json 2> gpurun_out/${T}_bench_cfg4.err; tail -1 gpurun_out/${T}_bench_cfg4.json | cut -c1-300
for c in 1 2 3; do
  timeout 600 python bench.py --config $c > gpurun_out/${T}_bench_cfg$c.json 2> gpurun_out/${T}_bench_cfg$c.err
  tail -1 gpurun_out/${T}_bench_cfg$c.json | cut -c1-200
done
timeout 600 python bench.py --sharded --no-cpu-baseline > gpurun_out/${T}_bench_cfg4_sharded.json 2> gpurun_out/${T}_bench_cfg4_sharded.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2>&1; tail -1 gpurun_out/${T}_bench_reference.json | cut -c1-200
PARITY_REPORT=gpurun_out/${T}_parity.json timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; tail -1 gpurun_out/${T}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_cfg4_launches.csv 2>/dev/null
for c in 4 1 2 3; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:acopf_tile_kernel -c 1 -o gpurun_out/${T}_cfg${c}_tile -f \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
done
