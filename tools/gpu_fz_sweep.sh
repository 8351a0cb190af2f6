mkdir -p gpurun_out
: > gpurun_out/fz_sweep.txt
for cfg in "12 4" "16 2" "16 1" "14 2" "12 2"; do set -- $cfg; echo "== WPB $1 CPP $2" >> gpurun_out/fz_sweep.txt; WPB=$1 CPP=$2 python tools/fused_prof.py 2>&1 | tail -5 >> gpurun_out/fz_sweep.txt; done
cat gpurun_out/fz_sweep.txt
