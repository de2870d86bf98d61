#!/bin/bash
# Round-2 end captures: cfg2 (launch list of the bench command + --set full of
# its four kernels), ePIE band/FFT kernels (cfg4) and evaluator kernels (cfg5).
out=gpurun_out; tag=${1:-r11}; mkdir -p $out
bash tools/profile_r2.sh $tag > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_cfg4_epie_launches.csv \
    python tools/prof_band.py cfg4 8 > /dev/null 2>&1
ncu --set full --clock-control none -k "regex:^(k|ke)" --launch-skip 40 -c 12 -o $out/${tag}_cfg4_epie \
    python tools/prof_band.py cfg4 8 > /dev/null 2>&1
ncu --set full --clock-control none -k "regex:kt2_fwd_rows|k_fwd_cols|ke_rows512|ke_cols512" -c 4 \
    -o $out/${tag}_eval python tools/prof_eval.py 64 > /dev/null 2>&1
for r in ${tag}_cfg4_epie ${tag}_eval; do
  ncu -i $out/$r.ncu-rep --page raw --csv > $out/${r}_raw.csv 2>/dev/null; rm -f $out/$r.ncu-rep
done
rm -f $out/*.ncu-rep
ls $out | grep $tag
