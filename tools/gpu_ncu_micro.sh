mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:spd_schur_w1" -c 1 -o gpurun_out/micro_w1 python tools/micro_bench.py 131072 > gpurun_out/ncu_micro_w1.log 2>&1
tail -3 gpurun_out/ncu_micro_w1.log
