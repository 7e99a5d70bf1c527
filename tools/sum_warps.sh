# Block-sum warps-per-CTA sweep (QCG_SUM_WARPS): parity tests, then C2 and C3 bench lines.
set -u
O=gpurun_out/sumw; mkdir -p $O
for w in 2 4 8; do
  QCG_SUM_WARPS=$w timeout 600 python -m pytest tests/test_gpu_statevector.py -m gpu -x -q -k "sum or expect" > $O/t$w.log 2>&1; echo "w=$w tests rc=$? $(tail -1 $O/t$w.log)"
done
for rep in 1 2; do
for w in 1 2 4 8; do
  QCG_SUM_WARPS=$w timeout 600 python bench.py --no-cpu-baseline > $O/c2_w$w.$rep.json 2> $O/c2_w$w.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_w$w.$rep.json').read().strip().splitlines()[-1]);print('c2 w=$w', round(d['ms_per_step'],2), d['step_ms'], round(d['roofline']['kernels']['blocksum']['ms'],3))"
done; done
for w in 1 2 4; do
  QCG_SUM_WARPS=$w timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > $O/c3_w$w.json 2> $O/c3_w$w.err
  python -c "import json,sys;d=json.loads(open('$O/c3_w$w.json').read().strip().splitlines()[-1]);print('c3 w=$w', round(d['ms_per_step'],2), d['step_ms'], round(d['roofline']['kernels']['blocksum']['ms'],3))"
done
