# ncu evidence for the bench command (small particle count keeps replays short).
# 1) launch list with device time per launch, 2) full capture of the top kernel.
set -x
CMD="python bench.py --steps 1 --warmup 3 --particles 2e6 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:logistic_abc -s 2 -c 2 -o gpurun_out/prof_logistic -f $CMD > gpurun_out/ncu_full.log 2>&1
CMD2="python scripts/time_kernels.py 2e6"
$CMD2 > gpurun_out/plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:logistic_abc -c 16 -o gpurun_out/prof_variants -f $CMD2 > gpurun_out/ncu_variants.log 2>&1
tail -n 3 gpurun_out/plain.log gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/ncu_variants.log
