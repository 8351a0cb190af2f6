mkdir -p gpurun_out
python tools/ds_bench.py | tail -1
python tools/micro_bench.py | tail -1
K=5 python tools/fused_big_bench.py | tail -1
timeout 1200 python -m pytest tests/test_struct_condense.py tests/test_gpu_condense.py tests/test_sd_tolerance.py tests/test_kernel_variants.py tests/test_boundary.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python bench.py --steps 50 --warmup 5 --no-micro --no-stokes --no-cfg3 --no-cpu-solver --cpu-sample 8 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'])"
