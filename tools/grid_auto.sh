# Auto grid (balanced when chunks share the GPU) vs forced full: C2 alternating, then the GPU suite.
set -u
O=gpurun_out/grida; mkdir -p $O
for rep in 1 2 3; do
for g in auto full; do
  if [ $g = auto ]; then unset QCG_GRID; else export QCG_GRID=$g; fi
  timeout 600 python bench.py --no-cpu-baseline > $O/c2_$g.$rep.json 2> $O/c2_$g.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_$g.$rep.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];print('c2 g=$g', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), round(k['pass_low']['ms'],2), round(k['pass_high']['ms'],2), round(d['roofline']['frac'],3), d['parity']['all_equal'] if 'parity' in d else '')"
done; done
unset QCG_GRID
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$? $(tail -1 $O/tests.log)"
