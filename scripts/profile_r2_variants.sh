# Round-2 ncu capture of the four instances of the fused logistic kernel and of the
# secondary kernels (one gpurun call; each ncu run follows a plain run that exited 0).
# The reports are summarised on the box (scripts/summarize_ncu.py) and removed: only the
# CSV summaries travel back (gpurun_out/ is capped at 64 MiB).
set -x
mkdir -p gpurun_out /tmp/vxbprof
CMD="python scripts/time_kernels.py 2e6"
$CMD > gpurun_out/r2_plain_variants.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:logistic_abc -c 16 -o /tmp/vxbprof/r2_prof_variants -f $CMD > gpurun_out/r2_ncu_variants.log 2>&1
python scripts/summarize_ncu.py /tmp/vxbprof/r2_prof_variants.ncu-rep gpurun_out/r2_ncu_full_logistic_variants
CMD2="python scripts/run_small_all.py"
$CMD2 > gpurun_out/r2_plain_small.log 2>&1 &&
ncu --set full --clock-control none -k "regex:ppp_kernel|abcsmc_propose|abcsmc_weights|tauleap_kernel|toggle_abc|anneal_kernel|tb_abc_kernel|radix_hist|accept_count" -c 40 -o /tmp/vxbprof/r2_prof_others -f $CMD2 > gpurun_out/r2_ncu_others.log 2>&1
python scripts/summarize_ncu.py /tmp/vxbprof/r2_prof_others.ncu-rep gpurun_out/r2_ncu_full_other_kernels
rm -rf /tmp/vxbprof
tail -n 3 gpurun_out/r2_plain_variants.log gpurun_out/r2_ncu_variants.log gpurun_out/r2_plain_small.log gpurun_out/r2_ncu_others.log
