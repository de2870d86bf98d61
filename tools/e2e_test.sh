python -m pytest tests/test_pft_gpu.py -q -m gpu -k "host_buffer" 2>&1 | tail -1
for mb in 16 32 64; do
PFTG_HOST_CHUNK_MB=$mb python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print('$mb', j["e2e"]["value"], j["e2e"]["two_calls_value"])'
done
