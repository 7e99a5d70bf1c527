set -u
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_blocksum' -c 2 \
    -o $O/sum_q20 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 > $O/sum_ncu.log 2>&1
tail -2 $O/sum_ncu.log
