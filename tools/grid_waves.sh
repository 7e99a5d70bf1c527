# Pass-kernel grid sweep (QCG_GRID = full | x2 | x3): parity tests, then C2 / C4 bench lines.
set -u
O=gpurun_out/gridw; mkdir -p $O
for g in x2 x3; do
  QCG_GRID=$g timeout 600 python -m pytest tests/test_gpu_statevector.py tests/test_gpu_large.py -m gpu -x -q > $O/t$g.log 2>&1; echo "g=$g tests rc=$? $(tail -1 $O/t$g.log)"
done
for rep in 1 2; do
for g in full x2 x3; do
  QCG_GRID=$g timeout 600 python bench.py --no-cpu-baseline > $O/c2_$g.$rep.json 2> $O/c2_$g.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_$g.$rep.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];print('c2 g=$g', round(d['ms_per_step'],2), d['step_ms'], round(k['pass_low']['ms'],2), round(k['pass_high']['ms'],2), round(d['roofline']['frac'],3))"
done; done
for g in full x2; do
  QCG_GRID=$g timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > $O/c4_$g.json 2> $O/c4_$g.err
  python -c "import json,sys;d=json.loads(open('$O/c4_$g.json').read().strip().splitlines()[-1]);print('c4 g=$g', round(d['ms_per_step'],2), d['step_ms'])"
done
