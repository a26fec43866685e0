# Launch list of one fixed-epsilon ABC step with early rejection (2e7 rows, the three kernel
# instances): the segment launches and what each costs.  Plain run first, then ncu.
set -x
mkdir -p gpurun_out
python scripts/early_reject_probe.py 2e7 > gpurun_out/r2_early_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:logistic_abc --csv --log-file gpurun_out/r2_launches_early_reject_2e7.csv \
    python scripts/early_reject_probe.py 2e7 > gpurun_out/r2_early_ncu.log 2>&1
tail -n 4 gpurun_out/r2_early_plain.log gpurun_out/r2_early_ncu.log
