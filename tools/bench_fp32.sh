# fp32-mode bench lines for the larger configs (outputs in gpurun_out/bench_*_fp32.json)
set -u
O=gpurun_out; mkdir -p $O
for w in c3 c4; do timeout 900 python bench.py --workload $w --precision 32 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_${w}_fp32.json 2> $O/bench_${w}_fp32.err; tail -c 150 $O/bench_${w}_fp32.json; echo; done
timeout 1500 python bench.py --workload c5 --precision 32 --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_c5_fp32.json 2> $O/bench_c5_fp32.err; tail -c 150 $O/bench_c5_fp32.json; echo
