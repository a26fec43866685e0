set -x
CMD="python scripts/run_small_all.py"
$CMD > gpurun_out/small_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'toggle_abc|tauleap|abcsmc_weights_fast|abcsmc_propose_fast' -c 16 -o gpurun_out/prof_others2 -f $CMD > gpurun_out/ncu_others2.log 2>&1
tail -n 5 gpurun_out/small_plain.log gpurun_out/ncu_others2.log
