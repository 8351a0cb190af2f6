mkdir -p gpurun_out
: > gpurun_out/amalg.txt
for a in "" "2-3" "1-2" "1-3" "1-2,3-4"; do
  echo "== MCS_AMALG='$a'" >> gpurun_out/amalg.txt
  MCS_AMALG="$a" python tools/coarse_bench.py 2 2>&1 | tail -2 >> gpurun_out/amalg.txt
  MCS_AMALG="$a" python tools/pcg_bench.py 10 2>&1 | tail -1 >> gpurun_out/amalg.txt
done
cat gpurun_out/amalg.txt
