# Refresh the committed bench lines on the GPU box (outputs in gpurun_out/bench_*.json).
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json; echo
timeout 600 python bench.py --impl reference > $O/bench_c2_ref.json 2> $O/bench_c2_ref.err; tail -c 200 $O/bench_c2_ref.json; echo
timeout 600 python bench.py --precision 32 --no-cpu-baseline > $O/bench_c2_fp32.json 2> $O/bench_c2_fp32.err
for w in c3 c4; do timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; tail -c 200 $O/bench_$w.json; echo; done
timeout 1500 python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 200 $O/bench_c5.json; echo
