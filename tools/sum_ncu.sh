# ncu capture of k_blocksum at a given subgraph size (Q, SLOTS env)
set -u
O=gpurun_out; mkdir -p $O
q=${QQ:-20}; s=${SLOTS:-21}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'k_blocksum' -c 1 \
    -o $O/sum_q$q python tools/pass_bench.py --q $q --slots $s --layers 1 --reps 1 > $O/sum_ncu.log 2>&1
tail -2 $O/sum_ncu.log
