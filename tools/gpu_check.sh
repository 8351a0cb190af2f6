# One GPU call: parity tests, bench line, launch list, full ncu capture of the hot kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
export MCS_NO_GRAPH=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-micro --cpu-sample 8 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:^(spd_schur_v5|condense_fused|elem_apply|ext_restrict|ext_prolong|jacobi_apply|mf_forward|mf_backward|mf_top_solve|cg_update)' -c 14 -o gpurun_out/full_${TAG:-r01} python tools/prof_kernels.py all > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
tail -3 gpurun_out/pytest_gpu.log
ls -la gpurun_out; du -sh gpurun_out
