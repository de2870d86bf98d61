for one in 1 0; do
  if [ $one = 1 ]; then export PFTG_EVAL_ONE_STREAM=1; else unset PFTG_EVAL_ONE_STREAM; fi
  python bench.py --workload cfg5 --steps 10 --warmup 3 2>&1 | grep '^{' | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print("one='$one'", j["ms_per_step"], {k: round(v/j["steps"],3) for k,v in j["roofline"]["kernel_ms"].items()})'
done
