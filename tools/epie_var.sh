for i in 1 2; do bash tools/epie_bench.sh v$i 2>&1 | grep json; done
