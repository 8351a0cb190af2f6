set -x
export MCS_NO_GRAPH=1
python tools/prof_kernels.py all > gpurun_out/pk.log 2>&1 || exit 1
PROF_IT=4 python tools/prof_pcg.py > gpurun_out/pp.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:^(spd_schur_v5|condense_v5|element_blocks|double_schur_v3|elem_apply|ext_restrict|ext_prolong|jacobi_apply|mf_forward|mf_backward|mf_top|csr_spmv|cg_update|dot_kernel|xpby|gather_sub|scatter)' -c 45 -o gpurun_out/full_r01b python tools/prof_kernels.py all > gpurun_out/ncu_full.log 2>&1
PROF_IT=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pcg_launches.csv python tools/prof_pcg.py > gpurun_out/ncu_pcg.log 2>&1
tail -2 gpurun_out/ncu_full.log gpurun_out/ncu_pcg.log
