mkdir -p gpurun_out
: > gpurun_out/ds_pf.txt
for v in 1 0; do echo "MCS_DSR_PF=$v" >> gpurun_out/ds_pf.txt; MCS_DSR_PF=$v timeout 300 python tools/ds_bench.py >> gpurun_out/ds_pf.txt 2>&1
MCS_DSR_PF=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k "regex:double_schur_reg" -c 1 python tools/ds_bench.py 2>&1 | grep -E "dram__|gpu__time" >> gpurun_out/ds_pf.txt; done
cat gpurun_out/ds_pf.txt
