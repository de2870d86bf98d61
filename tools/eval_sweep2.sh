#!/bin/bash
# evaluator chunk sweep (positions per FFT-chain chunk / per band-chain chunk), one or two streams
run() { env "$@" python bench.py --workload cfg5 --no-cpu-baseline --steps 5 2>&1 | tail -1 | python -c '
import json,sys
j=json.loads(sys.stdin.read()); print(sys.argv[1:], "ms/step %.3f" % j["ms_per_step"])' "$@"; }
run X=0
for c in 16 24 32 48 64 128; do run PFTG_EVAL_CHUNK=$c; done
for c in 32 64; do for p in 100 200 400; do run PFTG_EVAL_CHUNK=$c PFTG_EVAL_PCHUNK=$p; done; done
run PFTG_EVAL_ONE_STREAM=1 PFTG_EVAL_CHUNK=32
run PFTG_EVAL_ONE_STREAM=1 PFTG_EVAL_CHUNK=32 PFTG_EVAL_PCHUNK=32
