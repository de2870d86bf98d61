#!/bin/bash
# Rows-pass experiments on one B200 (run from the repo root): forward / adjoint
# rows kernels under the profiling switches; output -> gpurun_out/$1_exp.txt
tag=${1:-exp}
out=gpurun_out/${tag}_exp.txt
mkdir -p gpurun_out; : > $out
run() { echo "== $*" >> $out; env "$@" >> $out 2>&1; }
run python tools/fwd_only.py wide
run PFTG_NO_WIDE=1 python tools/fwd_only.py narrow
run PFTG_DEBUG_WS=1 python tools/fwd_only.py "wide groupB-idle"
run PFTG_DEBUG_WS=8 python tools/fwd_only.py "wide stageB-only"
run PFTG_DEBUG_WS=4 python tools/fwd_only.py "wide stageB+FFT"
run PFTG_TMA_NS=4 python tools/fwd_only.py "wide NS=4"
run PFTG_NO_WIDE=1 PFTG_DEBUG_WS=3 python tools/fwd_only.py "narrow stream-only"
run python tools/adj_only.py wide
run PFTG_NO_WIDE=1 python tools/adj_only.py narrow
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(kt|kc_)" -c 8 python tools/fwd_only.py >> $out 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(kt|kc_)" -c 4 python tools/adj_only.py >> $out 2>&1
