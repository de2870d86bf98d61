#!/bin/bash
# one-stream per-kernel times of the evaluator (clean isolated launches) + ncu of the eval_band kernels
out=gpurun_out; mkdir -p $out
for v in 3 0; do
  PFTG_EVAL_ONE_STREAM=1 PFTG_EVAL_BAND_OLD=$v python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | tail -1 | python -c '
import json,sys
j=json.loads(sys.stdin.read())
print("one-stream old=%s" % sys.argv[1], "ms/step %.3f" % j["ms_per_step"], {k: round(v,3) for k,v in j.get("roofline",{}).get("kernel_ms",{}).items() if v})' $v
done
ncu --set full --import-source on --clock-control none -k "regex:kb_rows|kb_cols|ke_rows512|ke_cols512" -c 4 -o $out/ebp python tools/prof_eval.py 64 > $out/ebp_ncu.log 2>&1
ncu -i $out/ebp.ncu-rep --page raw --csv > $out/ebp_raw.csv 2>/dev/null
ncu -i $out/ebp.ncu-rep --page source --csv --print-source sass --kernel-name regex:kb_rows > $out/ebp_rows_sass.csv 2>/dev/null
ncu -i $out/ebp.ncu-rep --page source --csv --print-source sass --kernel-name regex:kb_cols > $out/ebp_cols_sass.csv 2>/dev/null
rm -f $out/ebp.ncu-rep
python tools/raw_summary.py $out/ebp_raw.csv
