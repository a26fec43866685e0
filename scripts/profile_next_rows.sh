# ncu --set full of the SURVEY 8f kernels (toggle exact + throughput, annealed SMC, TB)
# after the same command exited 0 without ncu; summaries only (reports are too large).
set -x
CMD2="python scripts/run_small_all.py"
$CMD2 > gpurun_out/small_plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'anneal_kernel|tb_abc_kernel|toggle_abc' -c 8 -o gpurun_out/prof_next_v3 -f $CMD2 > gpurun_out/ncu_next3.log 2>&1
python scripts/summarize_ncu.py gpurun_out/prof_next_v3.ncu-rep gpurun_out/sum_next_v3
rm -f gpurun_out/prof_next_v3.ncu-rep
tail -n 4 gpurun_out/small_plain3.log
