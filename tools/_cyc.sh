python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | cut -c150-230
ACOPF_EXP_NO_AUX=1 python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | cut -c150-230
for n in noneP onlyA noA; do echo $n; ACOPF_EXP_NO_AUX=1 ACOPF_LIB_PATH=paper_2203_10587_b200/libexp_$n.so python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | cut -c150-230; done
