# Quick GPU check: parity tests, bench line, ncu full of the condensation kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
if [ -n "$NCU_K" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$NCU_K" -c ${NCU_C:-4} -o gpurun_out/${NCU_OUT:-quick} python tools/prof_kernels.py ${PROF_WHAT:-cfg} > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
fi
