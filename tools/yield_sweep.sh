# A/B of the FP64-pipe throttle masks (MCS_MICRO_YIELD, MCS_DS_YIELD)
mkdir -p gpurun_out
: > gpurun_out/yield_sweep.txt
for y in 0 1 2 4 8 5 6 9 10; do
  echo "MCS_MICRO_YIELD=$y" >> gpurun_out/yield_sweep.txt
  MCS_MICRO_YIELD=$y timeout 300 python tools/micro_bench.py >> gpurun_out/yield_sweep.txt 2>&1
done
for y in 0 1 2 3 4 5; do
  echo "MCS_DS_YIELD=$y" >> gpurun_out/yield_sweep.txt
  MCS_DS_YIELD=$y timeout 300 python tools/ds_bench.py >> gpurun_out/yield_sweep.txt 2>&1
done
cat gpurun_out/yield_sweep.txt
