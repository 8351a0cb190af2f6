# double Schur A/B: correctness (tests through mcs_double_schur) and time per variant
mkdir -p gpurun_out
: > gpurun_out/ds_ab.txt
for v in "MCS_DS=1" "MCS_DS=2" "MCS_DS=2 MCS_DSR_OCC=3" "MCS_DS=2 MCS_DSR_OCC=4"; do
  echo "== $v" >> gpurun_out/ds_ab.txt
  env $v timeout 300 python tools/ds_bench.py >> gpurun_out/ds_ab.txt 2>&1
done
echo "== tests with MCS_DS=2" >> gpurun_out/ds_ab.txt
MCS_DS=2 timeout 900 python -m pytest tests/test_sd_tolerance.py tests/test_gpu_condense.py tests/test_struct_condense.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15 >> gpurun_out/ds_ab.txt
cat gpurun_out/ds_ab.txt
