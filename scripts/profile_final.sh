# Round-1 ncu evidence (one B200).  Each capture runs only after the same command
# exited 0 without ncu.
set -x
CMD="python bench.py --steps 1 --warmup 3 --particles 2e6 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v2.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:logistic_abc -s 2 -c 2 -o gpurun_out/prof_logistic_v2 -f $CMD > gpurun_out/ncu_full.log 2>&1
CMD2="python scripts/run_small_all.py"
$CMD2 > gpurun_out/small_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'anneal_kernel|tb_abc_kernel|abcsmc_weights|ppp_kernel|tauleap_kernel|toggle_abc|abcsmc_propose' -c 24 -o gpurun_out/prof_others_v2 -f $CMD2 > gpurun_out/ncu_others.log 2>&1
tail -n 3 gpurun_out/plain.log gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/small_plain.log gpurun_out/ncu_others.log
# the reports are large: summarise on the box, keep only the CSVs (gpurun_out/ is capped at 64 MiB)
python scripts/summarize_ncu.py gpurun_out/prof_logistic_v2.ncu-rep gpurun_out/sum_logistic_v2
python scripts/summarize_ncu.py gpurun_out/prof_others_v2.ncu-rep gpurun_out/sum_others_v2
ncu -i gpurun_out/prof_logistic_v2.ncu-rep --page raw --csv > gpurun_out/raw_logistic_v2.csv
ncu -i gpurun_out/prof_logistic_v2.ncu-rep --page source --csv > gpurun_out/source_logistic_v2.csv 2>/dev/null
ls -la gpurun_out/*.ncu-rep
rm -f gpurun_out/prof_others_v2.ncu-rep
find gpurun_out -name 'prof_logistic_v2.ncu-rep' -size +30M -delete
# SURVEY 8f kernels (toggle, annealed SMC, TB)
$CMD2 > gpurun_out/small_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'anneal_kernel|tb_abc_kernel|toggle_abc' -c 6 -o gpurun_out/prof_next_v2 -f $CMD2 > gpurun_out/ncu_next.log 2>&1
python scripts/summarize_ncu.py gpurun_out/prof_next_v2.ncu-rep gpurun_out/sum_next_v2
rm -f gpurun_out/prof_next_v2.ncu-rep
# the three instances of the headline kernel
CMD3="python scripts/time_kernels.py 2e6"
$CMD3 > gpurun_out/plain_tk.log 2>&1 &&
ncu --set full --clock-control none -k regex:logistic_abc -c 10 -o gpurun_out/prof_variants_v2 -f $CMD3 > gpurun_out/ncu_tk.log 2>&1
python scripts/summarize_ncu.py gpurun_out/prof_variants_v2.ncu-rep gpurun_out/sum_variants_v2
rm -f gpurun_out/prof_variants_v2.ncu-rep
du -sh gpurun_out
