for n in base sp12 sp16 sp16t26 sp16t24; do
  if [ $n = base ]; then L=paper_2203_10587_b200/libacopf_b200.so; else L=paper_2203_10587_b200/libexp_$n.so; fi
  echo "$n: $(ACOPF_LIB_PATH=$L python bench.py --no-cpu-baseline --no-e2e --steps 20 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])') cfg4 $(ACOPF_LIB_PATH=$L python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
done
