set -x
python scripts/run_tb_small.py > gpurun_out/tb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tb_abc_kernel -s 1 -c 1 -o gpurun_out/prof_tb -f python scripts/run_tb_small.py > gpurun_out/ncu_tb.log 2>&1
python scripts/summarize_ncu.py gpurun_out/prof_tb.ncu-rep gpurun_out/sum_tb
ncu -i gpurun_out/prof_tb.ncu-rep --page source --csv > gpurun_out/source_tb.csv 2>/dev/null
ncu -i gpurun_out/prof_tb.ncu-rep --page details --csv > gpurun_out/details_tb.csv 2>/dev/null
rm -f gpurun_out/prof_tb.ncu-rep
tail -3 gpurun_out/tb_plain.log gpurun_out/ncu_tb.log
