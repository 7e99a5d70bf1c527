# Round-2 ncu evidence for the large-subgraph path: C3 launch list + full captures at
# q=24 (a7 pass A, v4 pass B, block sum) and q=26 (a7, TMA pass B b5, block sum).
set -u
O=gpurun_out/ncu2; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c3.csv \
    python bench.py --workload c3 --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu_c3.log 2>&1; echo "c3 list rc=$?"
python profiles/launch_summary.py $O/launches_c3.csv > $O/launch_summary_c3.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_pass|k_blocksum' -c 7 \
    -o $O/full_q24 python tools/pass_bench.py --q 24 --slots 4 --layers 1 --reps 1 > $O/ncu_full_q24.log 2>&1; echo "q24 rc=$?"
python profiles/ncu_stalls.py $O/full_q24.ncu-rep > $O/full_q24_summary.txt 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'k_pass|k_blocksum' -c 7 \
    -o $O/full_q26 python tools/pass_bench.py --q 26 --slots 2 --layers 1 --reps 1 > $O/ncu_full_q26.log 2>&1; echo "q26 rc=$?"
python profiles/ncu_stalls.py $O/full_q26.ncu-rep > $O/full_q26_summary.txt 2>&1
cat $O/full_q24_summary.txt $O/full_q26_summary.txt; tail -8 $O/launch_summary_c3.txt
