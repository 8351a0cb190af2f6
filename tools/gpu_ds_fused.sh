# double Schur + fused kernel iteration: parity tests, per-phase clocks, DS time, short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_struct_condense.py tests/test_gpu_condense.py tests/test_sd_tolerance.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/ds_bench.py 2>&1 | tail -1
python tools/fused_prof.py 2>&1 | tail -6
python bench.py --steps 20 --warmup 3 --no-micro --no-stokes --no-cfg3 --no-cpu-solver --cpu-sample 8 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'exec',d['roofline']['executed_frac'])
"
