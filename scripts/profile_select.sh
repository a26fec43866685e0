# ncu --set full of the six radix-select digit passes at 1e8 rows (after the same
# command exited 0 without ncu); only the summary leaves the box.
set -x
python scripts/time_select.py > gpurun_out/select_plain.log 2>&1 &&
ncu --set full --clock-control none -k regex:'radix_hist|count_valid' -s 21 -c 7 -o gpurun_out/prof_select -f python scripts/time_select.py > gpurun_out/ncu_select.log 2>&1
python scripts/summarize_ncu.py gpurun_out/prof_select.ncu-rep gpurun_out/sum_select
rm -f gpurun_out/prof_select.ncu-rep
tail -n 3 gpurun_out/select_plain.log
