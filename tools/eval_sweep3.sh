#!/bin/bash
run() { env "$@" python bench.py --workload cfg5 --no-cpu-baseline --steps 10 2>&1 | tail -1 | python -c '
import json,sys
j=json.loads(sys.stdin.read()); print(sys.argv[1:], "ms/step %.3f" % j["ms_per_step"])' "$@"; }
run X=0
for c in 200 400 800 1600; do run PFTG_EVAL_CHUNK=$c; done
for p in 200 400 1600; do run PFTG_EVAL_PCHUNK=$p; done
run PFTG_EVAL_CHUNK=800 PFTG_EVAL_PCHUNK=1600
run PFTG_EVAL_CHUNK=1600 PFTG_EVAL_PCHUNK=1600
run PFTG_EVAL_CHUNK=1600 PFTG_EVAL_PCHUNK=1600 PFTG_EVAL_ONE_STREAM=1
