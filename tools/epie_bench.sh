python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/${1}_cfg3.json
python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/${1}_cfg4.json
for w in cfg3 cfg4; do python -c 'import json,sys; j=json.load(open(sys.argv[1])); print(sys.argv[1], j["value"], j["band_updates_per_s"], j["fft_updates_per_s"], j["final_rel_err_aligned"], j["gpu_launches"])' gpurun_out/${1}_$w.json; done
