#!/bin/bash
tag=${1:-exp}
out=gpurun_out/${tag}_adjcols.txt
mkdir -p gpurun_out; : > $out
for d in 0 1 2 4 8 15; do echo "== dbg $d" >> $out; PFTG_DEBUG_ADJCOLS=$d python tools/adj_only.py "dbg $d" >> $out 2>&1; done
