#!/bin/bash
# A/B of the evaluator band chain (eval_band.cu): PFTG_EVAL_BAND_OLD bit 0 = batched rows kernel, bit 1 = generic cols kernel
for v in 3 2 1 0; do
  PFTG_EVAL_BAND_OLD=$v python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | tail -1 | python -c '
import json,sys
j=json.loads(sys.stdin.read())
print("old=%s" % sys.argv[1], "ms/step %.3f" % j["ms_per_step"], "phi_band %.9e" % j["phi_band"], "phi_fft %.9e" % j["phi_fft"], {k: round(v,3) for k,v in j.get("roofline",{}).get("kernel_ms",{}).items() if v})' $v
done
