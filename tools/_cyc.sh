tools/gpu_cycle.sh s10
ACOPF_LIB_PATH=paper_2203_10587_b200/libacopf_b200_m16.so python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | cut -c1-300
