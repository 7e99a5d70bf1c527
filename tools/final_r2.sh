# Round-2 final refresh at HEAD: GPU suite, smoke, both bench arms on C2, C1/C3/C4/C5 lines
# with their sampled reference CPU baselines, the fp32 C2 line, then the C2 launch list and
# one ncu --set full capture of the pass kernels.
set -u
O=gpurun_out/final; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)"
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 1500 python bench.py --impl reference > $O/bench_c2_ref.json 2> $O/bench_c2_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --precision 32 --no-cpu-baseline > $O/bench_c2_fp32.json 2> $O/bench_c2_fp32.err; echo "fp32 rc=$?"
timeout 900 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1 rc=$?"
for w in c3 c4; do timeout 1500 python bench.py --workload $w --steps 3 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; echo "$w rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu list rc=$?"
python profiles/launch_summary.py $O/launches.csv > $O/launch_summary.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_pass|k_blocksum' -c 5 \
    -o $O/full_c2 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python profiles/ncu_stalls.py $O/full_c2.ncu-rep > $O/full_c2_summary.txt 2>&1
timeout 2400 python bench.py --workload c5 --steps 1 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'), (d.get('parity') or {}).get('all_equal'))
"; done
