python -m pytest tests/test_ops_gpu.py tests/test_aux_gpu.py -q -x -m gpu 2>&1 | tail -3
bash tools/epie_bench.sh ${1:-p2}
