# Launch list of one C2 bench step + full ncu captures of the pass kernels (C2 chunk shape).
set -u
O=gpurun_out; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_pass|k_blocksum' -c 5 \
    -o $O/full_c2 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 > $O/ncu_full.log 2>&1
python profiles/ncu_stalls.py $O/full_c2.ncu-rep > $O/full_c2_summary.txt 2>&1
python profiles/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
cat $O/full_c2_summary.txt; tail -20 $O/launch_summary.txt
