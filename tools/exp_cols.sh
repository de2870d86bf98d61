#!/bin/bash
# Forward cols pass experiments (cfg2, 64 fields): grid size and profiling switches.
tag=${1:-exp}
out=gpurun_out/${tag}_cols.txt
mkdir -p gpurun_out; : > $out
run() { echo "== $*" >> $out; env "$@" >> $out 2>&1; }
run python tools/fwd_only.py base
for g in 148 222 444 592; do run PFTG_COLS_GRID=$g python tools/fwd_only.py "grid $g"; done
for d in 1 2 4 7; do run PFTG_DEBUG_COLS=$d python tools/fwd_only.py "dbg $d"; done
run PFTG_NO_PDL=1 python tools/fwd_only.py "no PDL"
run PFTG_NO_PDL=1 PFTG_DEBUG_COLS=7 python tools/fwd_only.py "no PDL dbg 7"
