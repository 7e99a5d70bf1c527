# ncu --set full capture of the TMA pass A at the C2 shape (gpurun_out/a5_q20.ncu-rep)
set -u
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_pass_a5' -c 3 \
    -o $O/a5_q20 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 > $O/a5_ncu.log 2>&1
tail -2 $O/a5_ncu.log
