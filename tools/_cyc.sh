ACOPF_LIB_PATH=paper_2203_10587_b200/libexp_mixed.so python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
echo "base: $(python bench.py --no-cpu-baseline --no-e2e --steps 20 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
echo "mixed: $(ACOPF_LIB_PATH=paper_2203_10587_b200/libexp_mixed.so python bench.py --no-cpu-baseline --no-e2e --steps 20 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
done
echo "mixed cfg4: $(ACOPF_LIB_PATH=paper_2203_10587_b200/libexp_mixed.so python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
