# Round evidence in one call: full GPU tests, smoke, bench (default), launch
# list of the bench, ncu --set full of the hot kernels.  TAG=<name>
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
if [ -n "$NCU" ]; then
export MCS_NO_GRAPH=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-micro --no-stokes --no-cfg3 --no-cpu-solver --cpu-sample 8 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:(condense_fused|spd_schur_w1|elem_apply|ext_restrict|ext_prolong|jacobi_apply|mf_forward|mf_top_solve|cg_update)" -c 12 -o gpurun_out/full_$TAG python tools/prof_kernels.py all > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:(condense_fused_kernel|double_schur_reg)" -c 2 -o gpurun_out/full_ds_$TAG python tools/prof_kernels.py ds > gpurun_out/ncu_full_ds_$TAG.log 2>&1
# summarise on the box; the full-size cfg3 report is too large to bring back (64 MiB limit)
python tools/ncu_summary.py gpurun_out/ncu_kernels_$TAG gpurun_out/full_$TAG.ncu-rep gpurun_out/full_ds_$TAG.ncu-rep > gpurun_out/ncu_summary_$TAG.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_bench_$TAG.txt 2>&1
rm -f gpurun_out/full_ds_$TAG.ncu-rep
fi
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; tail -2 gpurun_out/bench_$TAG.err
