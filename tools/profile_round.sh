#!/bin/bash
# Profile artifacts for one round (run on the GPU box from the repo root):
#   1. the default bench line (no profiler),
#   2. the ncu launch list of the same command (per-launch gpu__time_duration),
#   3. one `--set full` capture of the dominant kernel (first forward rows pass launch).
# Usage: tools/profile_round.sh TAG   -> gpurun_out/TAG_*
set -e
tag=${1:-round}
out=gpurun_out
mkdir -p $out
python bench.py > $out/${tag}_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(k_|kf_|kt|kc_)" --csv \
    --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:kt2_fwd_rows" -c 1 \
    -o $out/${tag}_rows_fwd python tools/prof_pft.py > $out/${tag}_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:kt_adj_rows" -c 1 \
    -o $out/${tag}_rows_adj python tools/prof_pft.py > $out/${tag}_ncu_full_adj.log 2>&1
# export summaries on the box (the .ncu-rep files are too large to bring back whole)
for k in rows_fwd rows_adj; do
  ncu -i $out/${tag}_$k.ncu-rep --page raw --csv > $out/${tag}_${k}_raw.csv 2>/dev/null || true
  ncu -i $out/${tag}_$k.ncu-rep --page details --csv > $out/${tag}_${k}_details.csv 2>/dev/null || true
  ncu -i $out/${tag}_$k.ncu-rep --page source --csv --print-source sass > $out/${tag}_${k}_sass.csv 2>/dev/null || true
done
ls -la $out
[ -n "$KEEP_REP" ] || rm -f $out/${tag}_rows_adj.ncu-rep
echo done
