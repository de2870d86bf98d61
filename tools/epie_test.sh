timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_facade_gpu.py tests/test_aux_gpu.py -q -x -m gpu -rf 2>&1 | tail -3
for v in "" "PFTG_NO_PERSIST=1"; do
for w in cfg3 cfg4; do
  env $v timeout 300 python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep '^{' | python -c 'import json,sys,statistics; j=json.loads(sys.stdin.read()); sw=j["sweep_ms"]; pb=j["config"]["pft_sweeps"]; print("'$w' '$v'", round(j["value"]), round(j["band_updates_per_s"]), round(j["fft_updates_per_s"]), round(statistics.median(sw[1:pb]),2), "ms/band sweep", j["final_rel_err_aligned"])'
done; done
