#!/bin/bash
# Chunking / L2-hint experiments for the cfg2 forward and adjoint passes.
tag=${1:-exp}
out=gpurun_out/${tag}_chunks.txt
mkdir -p gpurun_out; : > $out
run() { echo "== $*" >> $out; env "$@" >> $out 2>&1; }
run python tools/fwd_only.py "24MB balanced"
run PFTG_DEBUG_WS=16 python tools/fwd_only.py "24MB balanced, no L2 hint"
run PFTG_CHUNK_MB=48 python tools/fwd_only.py "48MB (1 chunk)"
run PFTG_CHUNK_MB=48 PFTG_DEBUG_WS=16 python tools/fwd_only.py "48MB no hint"
run PFTG_DEBUG_WS=1 python tools/fwd_only.py "groupB idle"
run PFTG_CHUNK_MB=48 PFTG_DEBUG_WS=1 python tools/fwd_only.py "48MB groupB idle"
run python tools/adj_only.py "24MB"
run PFTG_CHUNK_MB=48 python tools/adj_only.py "48MB"
python bench.py --no-cpu-baseline >> $out 2>&1
PFTG_CHUNK_MB=48 python bench.py --no-cpu-baseline >> $out 2>&1
