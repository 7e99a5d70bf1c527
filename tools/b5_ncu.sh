# ncu --set full captures of pass B (TMA and v4) at the C2 shape
set -u
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_pass_b' -c 4 \
    -o $O/b5_q20 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 > $O/b5_ncu.log 2>&1
QCG_PASS_B=v4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_pass_b' -c 4 \
    -o $O/v4b_q20 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 >> $O/b5_ncu.log 2>&1
tail -3 $O/b5_ncu.log
