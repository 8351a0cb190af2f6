mkdir -p gpurun_out
: > gpurun_out/micro_pf.txt
for v in 1 0; do echo "MCS_MICRO_PF=$v" >> gpurun_out/micro_pf.txt; MCS_MICRO_PF=$v timeout 300 python tools/micro_bench.py >> gpurun_out/micro_pf.txt 2>&1
MCS_MICRO_PF=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:spd_schur_w1" -c 1 python tools/micro_bench.py 131072 2>&1 | grep -E "dram__|gpu__time" >> gpurun_out/micro_pf.txt; done
cat gpurun_out/micro_pf.txt
