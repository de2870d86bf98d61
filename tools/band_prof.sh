ncu --set full --import-source on --clock-control none --cache-control none -k "regex:k_fwd_cols|kf_adj_rows" --launch-skip 8 -c 4 -o gpurun_out/b1_band python tools/prof_band.py cfg4 8 > /dev/null 2>&1
ncu -i gpurun_out/b1_band.ncu-rep --page raw --csv > gpurun_out/b1_band_raw.csv
for k in k_fwd_cols kf_adj_rows; do ncu -i gpurun_out/b1_band.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/b1_src_$k.csv 2>/dev/null; done
python tools/raw_summary.py gpurun_out/b1_band_raw.csv; rm -f gpurun_out/b1_band.ncu-rep
