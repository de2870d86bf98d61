#!/bin/bash
# All bench workloads + the reference arm, one line each -> gpurun_out/TAG_results.txt
tag=${1:-round}
out=gpurun_out/${tag}_results.txt
mkdir -p gpurun_out; : > $out
timeout 400 python bench.py >> $out 2>gpurun_out/${tag}_err_cfg2.log
for w in cfg1 cfg3 cfg5; do timeout 600 python bench.py --workload $w >> $out 2>gpurun_out/${tag}_err_$w.log; done
timeout 900 python bench.py --workload cfg4 --steps 1 --warmup 1 >> $out 2>gpurun_out/${tag}_err_cfg4.log
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 >> $out 2>gpurun_out/${tag}_err_ref.log
