for i in 1 2; do python bench.py --workload cfg5 --steps 10 --warmup 3 2>&1 | grep '^{' | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["ms_per_step"], j["value"], j["phi_fft"], j["phi_band"])'; done
python -m pytest tests/test_ops_gpu.py tests/test_dist.py -q -m gpu -k "evaluator or evaluate" 2>&1 | tail -1
