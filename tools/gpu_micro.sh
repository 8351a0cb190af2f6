mkdir -p gpurun_out
: > gpurun_out/micro_ab.txt
for v in 2 3 1; do echo "MCS_MICRO=$v" >> gpurun_out/micro_ab.txt; MCS_MICRO=$v timeout 300 python tools/micro_bench.py >> gpurun_out/micro_ab.txt 2>&1; done
for v in 0 1; do echo "MCS_DSR_PAIR=$v" >> gpurun_out/micro_ab.txt; MCS_DSR_PAIR=$v timeout 300 python tools/ds_bench.py >> gpurun_out/micro_ab.txt 2>&1; done
cat gpurun_out/micro_ab.txt
bash tools/gpu_ds_fused.sh
