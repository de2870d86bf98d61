#!/bin/bash
# Round-2 results: new full-size tests, every workload's bench line (with CPU baselines).
out=gpurun_out; mkdir -p $out; tag=${1:-r10}
python -m pytest tests/test_pft_gpu.py tests/test_ops_gpu.py -q -m gpu -k "full_cfg2_size or cfg5_full_size" 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 > $out/${tag}_bench_cfg2.log 2>&1
for w in cfg1 cfg3 cfg5; do python bench.py --workload $w --steps 10 --warmup 3 > $out/${tag}_bench_$w.log 2>&1; done
python bench.py --workload cfg4 --steps 10 --warmup 3 > $out/${tag}_bench_cfg4.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $out/${tag}_bench_ref.log 2>&1
for w in cfg1 cfg2 cfg3 cfg4 cfg5 ref; do tail -1 $out/${tag}_bench_$w.log | cut -c1-400; echo; done
