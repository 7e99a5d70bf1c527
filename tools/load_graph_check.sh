# Parallel graph validation (load_graph): GPU suite, then C4 / C2 end-to-end lines.
set -u
O=gpurun_out/lg; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$? $(tail -1 $O/tests.log)"
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/c4.json 2> $O/c4.err
python -c "import json;d=json.loads(open('$O/c4.json').read().strip().splitlines()[-1]);print('c4', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['e2e']['step_ms'], d['e2e'].get('stage_s'))"
timeout 600 python bench.py --no-cpu-baseline > $O/c2.json 2> $O/c2.err
python -c "import json;d=json.loads(open('$O/c2.json').read().strip().splitlines()[-1]);print('c2', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"
