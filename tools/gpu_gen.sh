mkdir -p gpurun_out
: > gpurun_out/gen_ab.txt
for K in 6 5; do for G in 1 2; do K=$K MCS_GEN=$G timeout 300 python tools/gen_bench.py >> gpurun_out/gen_ab.txt 2>&1; done; done
cat gpurun_out/gen_ab.txt
timeout 900 python -m pytest tests/test_struct_condense.py tests/test_gpu_condense.py tests/test_sd_tolerance.py tests/test_full_size.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
