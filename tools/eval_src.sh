ncu --set full --import-source on --clock-control none -k "regex:kt2_fwd_rows|k_fwd_cols|ke_rows512|ke_cols512" -c 4 -o gpurun_out/s1_eval python tools/prof_eval.py 64 > gpurun_out/s1_ncu.log 2>&1
for k in kt2_fwd_rows k_fwd_cols ke_rows512 ke_cols512_eval; do
  ncu -i gpurun_out/s1_eval.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/s1_src_$k.csv 2>/dev/null
done
ls -la gpurun_out/ | grep s1_
