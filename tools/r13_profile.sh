#!/bin/bash
# Round-2 end captures (r13): cfg2 (launch list of the bench command + --set full of its
# four kernels), ePIE band-stage kernels of eval_band.cu (cfg4), evaluator kernels (cfg5,
# one 64-position chunk).
out=gpurun_out; tag=${1:-r13}; mkdir -p $out
bash tools/profile_r2.sh $tag > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_cfg4_epie_launches.csv \
    python tools/prof_band.py cfg4 8 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k "regex:kb_|ke_epie" --launch-skip 8 -c 9 -o $out/${tag}_cfg4_epie \
    python tools/prof_band.py cfg4 8 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k "regex:kb_rows|kb_cols|ke_rows512|ke_cols512" -c 4 \
    -o $out/${tag}_eval python tools/prof_eval.py 64 > /dev/null 2>&1
for r in ${tag}_cfg4_epie ${tag}_eval; do
  ncu -i $out/$r.ncu-rep --page raw --csv > $out/${r}_raw.csv 2>/dev/null
done
ncu -i $out/${tag}_eval.ncu-rep --page source --csv --print-source sass --kernel-name regex:kb_rows > $out/${tag}_kb_rows_sass.csv 2>/dev/null
ncu -i $out/${tag}_cfg4_epie.ncu-rep --page source --csv --print-source sass --kernel-name regex:kb_adj_rows --launch-count 1 > $out/${tag}_kb_adj_rows_sass.csv 2>/dev/null
rm -f $out/*.ncu-rep
bash tools/round_results.sh $tag
ls $out | grep $tag
