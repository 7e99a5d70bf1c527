# Full GPU tests + C3/C5 fp64 bench lines (outputs in gpurun_out/)
set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python -c "import json;d=json.loads(open('$O/bench_c3.json').readline());print('c3', round(d['ms_per_step'],1), d['clocks']['reasons'])"
timeout 1500 python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
python -c "import json;d=json.loads(open('$O/bench_c5.json').readline());print('c5', round(d['ms_per_step'],1), d['clocks']['reasons'])"
