#!/bin/bash
# Round-2 baseline on the GPU box: tests, every workload's bench line, and ncu
# evidence for the evaluator (cfg5) and ePIE (cfg3/cfg4) kernels.
out=gpurun_out; mkdir -p $out; tag=${1:-r8}
python -m pytest tests -m gpu -q --timeout 600 -rf > $out/${tag}_tests.log 2>&1
tail -3 $out/${tag}_tests.log
python bench.py --steps 20 --warmup 5 > $out/${tag}_bench_cfg2.log 2>&1
for w in cfg1 cfg3 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 > $out/${tag}_bench_$w.log 2>&1; done
python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline > $out/${tag}_bench_cfg4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_eval_launches.csv \
    python tools/prof_eval.py 64 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k "regex:kt2_fwd_rows|k_fwd_cols|ke_rows512|ke_cols512" -c 4 \
    -o $out/${tag}_eval python tools/prof_eval.py 64 > $out/${tag}_ncu_eval.log 2>&1
for c in cfg3 cfg4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_${c}_epie_launches.csv \
      python tools/prof_band.py $c 8 > /dev/null 2>&1
  ncu --set full --import-source on --clock-control none -k "regex:^(k|ke)" --launch-skip 40 -c 14 \
      -o $out/${tag}_${c}_epie python tools/prof_band.py $c 8 > $out/${tag}_ncu_${c}.log 2>&1
done
for r in $out/${tag}_eval $out/${tag}_cfg3_epie $out/${tag}_cfg4_epie; do
  ncu -i $r.ncu-rep --page raw --csv > ${r}_raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details --csv > ${r}_details.csv 2>/dev/null
done
rm -f $out/*.ncu-rep
ls -la $out | tail -30
