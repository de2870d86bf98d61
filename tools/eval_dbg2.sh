export PFTG_LIB_PATH=$PWD/paper_2408_03532_b200/prof/libpftg.so PFTG_EVAL_ONE_STREAM=1 PFTG_DEBUG_WS=1
ncu --set full --clock-control none -k "regex:kt2_fwd_rows" -c 1 -o gpurun_out/d2_kt2_groupA python tools/prof_eval.py 64 > /dev/null 2>&1
ncu -i gpurun_out/d2_kt2_groupA.ncu-rep --page raw --csv > gpurun_out/d2_kt2_groupA_raw.csv
ncu -i gpurun_out/d2_kt2_groupA.ncu-rep --page details --csv > gpurun_out/d2_kt2_groupA_details.csv
python tools/raw_summary.py gpurun_out/d2_kt2_groupA_raw.csv
