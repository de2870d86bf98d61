ncu --set full --import-source on --clock-control none --cache-control none -k "regex:kq_" -c 6 -o gpurun_out/tq python tools/cfg1_prof.py > /dev/null 2>&1
for k in kq_fwd_ab kq_adj_band kq_adj_ab kq_fft2 kq_band; do ncu -i gpurun_out/tq.ncu-rep --page source --csv --print-source sass -k regex:$k -c 1 > gpurun_out/tq_src_$k.csv 2>/dev/null; done
ncu -i gpurun_out/tq.ncu-rep --page raw --csv > gpurun_out/tq_raw.csv
rm -f gpurun_out/tq.ncu-rep
python tools/raw_summary.py gpurun_out/tq_raw.csv
