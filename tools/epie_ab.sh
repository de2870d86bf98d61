#!/bin/bash
# ePIE band stage A/B: PFTG_EVAL_BAND_OLD bits (4 = generic cols, 8 = streaming adjoint rows), PFTG_NO_PERSIST
run() { w=$1; shift; env "$@" python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep "^{" | python -c '
import json,sys
j=json.loads(sys.stdin.read()); print(sys.argv[1:], "%.0f band %.0f fft %.0f err %.4f obj %.3f launches %d" % (j["value"], j["band_updates_per_s"], j["fft_updates_per_s"], j["final_rel_err_aligned"], j["final_objective"], j["gpu_launches"]))' $w "$@"; }
run cfg4 PFTG_EVAL_BAND_OLD=12
run cfg4 PFTG_EVAL_BAND_OLD=8
run cfg4 PFTG_EVAL_BAND_OLD=0
run cfg3 PFTG_EVAL_BAND_OLD=12
run cfg3 PFTG_EVAL_BAND_OLD=0
run cfg3 PFTG_EVAL_BAND_OLD=0 PFTG_NO_PERSIST=1
