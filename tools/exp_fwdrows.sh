#!/bin/bash
tag=${1:-exp}
out=gpurun_out/${tag}_fwdrows.txt
mkdir -p gpurun_out; : > $out
for d in 0 1 8 4 32; do echo "== PFTG_DEBUG_WS=$d" >> $out; PFTG_DEBUG_WS=$d python tools/fwd_only.py "dbg $d" >> $out 2>&1; done
