# Round-2 final ncu capture of the workload kernels besides the fused logistic kernel:
# tau-leap (exact / throughput / fp32 instances), toggle (both instances), annealed SMC,
# TB Gillespie and the ABC-SMC weights -- the plain run first, the summary made on the box.
set -x
mkdir -p gpurun_out /tmp/vxbprof
CMD="python scripts/run_small_all.py"
$CMD > gpurun_out/r2_plain_small_final.log 2>&1 &&
ncu --set full --clock-control none -k "regex:tauleap|toggle_abc|anneal_kernel|tb_abc_kernel|abcsmc_weights" -c 40 -o /tmp/vxbprof/r2_prof_final -f $CMD > gpurun_out/r2_ncu_final.log 2>&1
python scripts/summarize_ncu.py /tmp/vxbprof/r2_prof_final.ncu-rep gpurun_out/r2_ncu_full_workload_kernels
rm -rf /tmp/vxbprof
tail -n 3 gpurun_out/r2_plain_small_final.log gpurun_out/r2_ncu_final.log
