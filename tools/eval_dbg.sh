# kt2_fwd_rows time split in the evaluator (cfg5), profiling build: group B idle (1),
# stage B only (8), stage B + FFT (4), band staged without G stores (32), full (0)
export PFTG_LIB_PATH=$PWD/paper_2408_03532_b200/prof/libpftg.so PFTG_EVAL_ONE_STREAM=1
for d in 0 1 8 4 32; do
  PFTG_DEBUG_WS=$d python bench.py --workload cfg5 --steps 5 --warmup 3 2>&1 | grep '^{' | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print("dbg='$d'", {k: round(v/j["steps"],3) for k,v in j["roofline"]["kernel_ms"].items() if v})'
done
