# ncu evidence for the large-subgraph path: C3 launch list + full captures at q=24
set -u
O=gpurun_out; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c3.csv \
    python bench.py --workload c3 --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu_c3.log 2>&1
python profiles/launch_summary.py $O/launches_c3.csv > $O/launch_summary_c3.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_pass|k_blocksum' -c 5 \
    -o $O/full_q24 python tools/pass_bench.py --q 24 --slots 4 --layers 1 --reps 1 > $O/ncu_full_q24.log 2>&1
python profiles/ncu_stalls.py $O/full_q24.ncu-rep > $O/full_q24_summary.txt 2>&1
cat $O/full_q24_summary.txt; cat $O/launch_summary_c3.txt
