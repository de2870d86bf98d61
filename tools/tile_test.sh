./tools/cfg1_time
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/t10_tile.csv python tools/cfg1_prof.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t10_empty.csv ./tools/empty_kernel > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/t10_tile.csv; python tools/launch_summary.py gpurun_out/t10_empty.csv
