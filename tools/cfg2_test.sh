python -m pytest tests/test_pft_gpu.py -q -x -m gpu 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["ms_per_step"], j["value"], {k: round(v/j["steps"]*1e3,2) for k,v in j["roofline"]["kernel_ms"].items() if v})'; done
