# ncu --set full of the kernels reworked late in round 2: the tau-leap instances on ALL six
# levels (levels 4-5 are the quiet regime that config 4's time is made of) and the segment
# launches of early rejection.  Plain runs first; summaries made on the box.
set -x
mkdir -p gpurun_out /tmp/vxbprof
CMD="python scripts/run_tauleap_all_levels.py 40000"
$CMD > gpurun_out/r2_plain_tl.log 2>&1 &&
ncu --set full --clock-control none -k regex:tauleap -c 18 -o /tmp/vxbprof/r2_tl -f $CMD > gpurun_out/r2_ncu_tl.log 2>&1
python scripts/summarize_ncu.py /tmp/vxbprof/r2_tl.ncu-rep gpurun_out/r2_ncu_full_tauleap_all_levels
CMD2="python scripts/early_reject_probe.py 2e6"
$CMD2 > gpurun_out/r2_plain_er.log 2>&1 &&
ncu --set full --clock-control none -k regex:logistic_abc -c 40 -o /tmp/vxbprof/r2_er -f $CMD2 > gpurun_out/r2_ncu_er.log 2>&1
python scripts/summarize_ncu.py /tmp/vxbprof/r2_er.ncu-rep gpurun_out/r2_ncu_full_early_reject_segments
rm -rf /tmp/vxbprof
tail -n 3 gpurun_out/r2_plain_tl.log gpurun_out/r2_plain_er.log
