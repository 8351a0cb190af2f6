mkdir -p gpurun_out
bash tools/gpu_ds_fused.sh
K=5 python tools/gen_bench.py
timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_gpu_pcg.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
