#!/bin/bash
# Round profile: bench line, launch list of the bench command, --set full of the
# four cfg2 kernels (first launch of each in tools/prof_pft.py). -> gpurun_out/TAG_*
set -e
tag=${1:-round}
out=gpurun_out
mkdir -p $out
python bench.py > $out/${tag}_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(k_|kf_|kt|kc_)" --csv \
    --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1
for k in kt2_fwd_rows kc_fwd_cols_local kc_adj_cols_local kt_adj_rows; do
  ncu --set full --import-source on --clock-control none -k "regex:$k" -c 1 -o $out/${tag}_$k python tools/prof_pft.py > $out/${tag}_ncu_$k.log 2>&1 || true
  ncu -i $out/${tag}_$k.ncu-rep --page raw --csv > $out/${tag}_${k}_raw.csv 2>/dev/null || true
  ncu -i $out/${tag}_$k.ncu-rep --page details --csv > $out/${tag}_${k}_details.csv 2>/dev/null || true
  ncu -i $out/${tag}_$k.ncu-rep --page source --csv --print-source sass > $out/${tag}_${k}_sass.csv 2>/dev/null || true
  rm -f $out/${tag}_$k.ncu-rep
done
ls -la $out | grep $tag
echo done
