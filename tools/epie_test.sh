timeout 900 python -m pytest tests/test_ops_gpu.py -q -x -m gpu -rf 2>&1 | tail -1
for w in cfg3 cfg4; do
  timeout 300 python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep '^{' | python -c 'import json,sys,statistics; j=json.loads(sys.stdin.read()); sw=j["sweep_ms"]; pb=j["config"]["pft_sweeps"]; print("'$w'", round(j["value"]), round(j["band_updates_per_s"]), round(j["fft_updates_per_s"]), round(statistics.median(sw[1:pb]),2), round(statistics.median(sw[pb+1:]),2), "ms/band,fft sweep", j["final_rel_err_aligned"])'
done
