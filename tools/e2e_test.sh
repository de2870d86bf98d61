# e2e host pipeline: PCIe ceiling, host-buffer parity tests, bench e2e per chunk size
mkdir -p gpurun_out
./tools/pcie_probe 2>&1
python -m pytest tests -q -m gpu -k "host" 2>&1 | tail -1
for mb in ${E2E_MBS:-8 16 32}; do
PFTG_HOST_CHUNK_MB=$mb python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print('$mb', j["e2e"]["value"], j["e2e"]["two_calls_value"])'
done
