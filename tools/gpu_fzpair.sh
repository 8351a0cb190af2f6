for p in 0 1; do for K in 6 5; do MCS_FZ_PAIR=$p K=$K python tools/gen_bench.py 2>&1 | tail -1; done; done
