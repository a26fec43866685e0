# Round-2 ncu evidence (one gpurun call; every ncu run follows a plain run of the same
# command that exited 0).  1) launch list of the bench command, 2) full capture of the
# headline kernel, 3) full capture of the kernels added in round 2.
set -x
CMD="python bench.py --steps 1 --warmup 3 --particles 2e6 --no-extras"
$CMD > gpurun_out/r2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1
$CMD > gpurun_out/r2_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:logistic_abc -s 2 -c 2 -o gpurun_out/r2_prof_logistic -f $CMD > gpurun_out/r2_ncu_full.log 2>&1
CMD2="python scripts/run_new_kernels_r2.py"
$CMD2 > gpurun_out/r2_plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:seq_expsum|resample_draw|pack_rows|append_rows|append_state|chunk_total|max_partial" -c 24 -o gpurun_out/r2_prof_new -f $CMD2 > gpurun_out/r2_ncu_new.log 2>&1
tail -n 3 gpurun_out/r2_plain.log gpurun_out/r2_ncu_launch.log gpurun_out/r2_ncu_full.log gpurun_out/r2_plain3.log gpurun_out/r2_ncu_new.log
