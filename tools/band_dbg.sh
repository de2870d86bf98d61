# ePIE band-stage time split (profiling build): kf_adj_rows without P1 (1), without the
# fused stage B (2), without the epilogue (4); results invalid, timing only
export PFTG_LIB_PATH=$PWD/paper_2408_03532_b200/prof/libpftg.so
for d in 0 1 4 5 7; do
  for w in cfg3 cfg4; do
  PFTG_DEBUG_ADJ=$d python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep '^{' | python -c 'import json,sys,statistics; j=json.loads(sys.stdin.read()); sw=j["sweep_ms"]; pb=j["config"]["pft_sweeps"]; print("'$w' dbg='$d'", round(statistics.median(sw[1:pb]),2), "ms/band sweep", round(statistics.median(sw[pb+1:]),2), "ms/fft sweep")'
  done
done
