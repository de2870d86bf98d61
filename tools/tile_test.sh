./tools/cfg1_time; ./tools/cfg1_time
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/t11_tile.csv python tools/cfg1_prof.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/t11_tile.csv
python -m pytest tests/test_pft_gpu.py tests/test_golden_gpu.py tests/test_facade_gpu.py -q -x -m gpu 2>&1 | tail -1
