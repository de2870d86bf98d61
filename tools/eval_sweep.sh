#!/bin/bash
# Evaluator (cfg5) knob sweep: chunk size and one vs two streams.
out=gpurun_out; mkdir -p $out; tag=${1:-e1}
for c in 8 16 32; do
  for one in 0 1; do
    if [ $one = 1 ]; then export PFTG_EVAL_ONE_STREAM=1; else unset PFTG_EVAL_ONE_STREAM; fi
    echo "chunk=$c one_stream=$one $(PFTG_EVAL_CHUNK=$c python bench.py --workload cfg5 --steps 10 --warmup 3 2>&1 | grep '^{' | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["ms_per_step"], j["roofline"]["kernel_ms"])')"
  done
done > $out/${tag}_eval_sweep.txt 2>&1
unset PFTG_EVAL_ONE_STREAM
./tools/fma_peak > $out/${tag}_fma_peak.json 2>&1
cat $out/${tag}_eval_sweep.txt $out/${tag}_fma_peak.json
