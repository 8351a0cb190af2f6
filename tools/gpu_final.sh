# Round-end evidence: tests, smoke, bench lines (cfg2 default, cfg3), launch list,
# ncu --set full of the hot kernels (small capture), PCG launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --cfg 3 --steps 5 --warmup 3 --no-micro --no-stokes > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
export MCS_NO_GRAPH=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-micro --no-stokes --cpu-sample 8 > gpurun_out/ncu_launch.log 2>&1
PROF_IT=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg_launches.csv python tools/prof_pcg.py > gpurun_out/ncu_pcg.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:^(condense_fused|elem_apply|ext_restrict|ext_prolong|jacobi_apply|mf_forward|mf_top_solve|cg_update|spd_schur_v5)' -c 9 -o gpurun_out/full_final python tools/prof_kernels.py all > gpurun_out/ncu_full.log 2>&1
MCS_NO_GRAPH=1 PROF_COMP=additive timeout 300 ncu --set full --import-source on --clock-control none -k 'regex:^elem_apply' -c 1 -o gpurun_out/full_apply42 python tools/prof_kernels.py cfg > gpurun_out/ncu_apply42.log 2>&1
python tools/fused_prof.py > gpurun_out/fprof.txt 2>&1
du -sh gpurun_out
