for n in w3 w4; do echo "$n tests: $(ACOPF_LIB_PATH=paper_2203_10587_b200/libexp_$n.so python -m pytest tests -m gpu -x -q 2>&1 | tail -1)"; done
for i in 1 2; do for n in base w3 w4; do
  if [ $n = base ]; then L=paper_2203_10587_b200/libacopf_b200.so; else L=paper_2203_10587_b200/libexp_$n.so; fi
  echo "$n: $(ACOPF_LIB_PATH=$L python bench.py --no-cpu-baseline --no-e2e --steps 20 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
done; done
for n in base w3 w4; do
  if [ $n = base ]; then L=paper_2203_10587_b200/libacopf_b200.so; else L=paper_2203_10587_b200/libexp_$n.so; fi
  echo "$n cfg4: $(ACOPF_LIB_PATH=$L python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])') cfg2: $(ACOPF_LIB_PATH=$L python bench.py --config 2 --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
done
