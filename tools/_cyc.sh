python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2; do
echo "m12: $(python bench.py --no-cpu-baseline --no-e2e --steps 20 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
echo "m16: $(ACOPF_LIB_PATH=paper_2203_10587_b200/libacopf_b200_m16.so python bench.py --no-cpu-baseline --no-e2e --steps 20 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
done
echo "m16 cfg4: $(ACOPF_LIB_PATH=paper_2203_10587_b200/libacopf_b200_m16.so python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
echo "m12 cfg4: $(python bench.py --config 4 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
