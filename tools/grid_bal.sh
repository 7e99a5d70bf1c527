# QCG_GRID=bal vs full on C2 (a7 pass A), alternating runs.
set -u
O=gpurun_out/gridb; mkdir -p $O
for rep in 1 2 3; do
for g in full bal; do
  QCG_GRID=$g timeout 600 python bench.py --no-cpu-baseline > $O/c2_$g.$rep.json 2> $O/c2_$g.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_$g.$rep.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];print('c2 g=$g', round(d['ms_per_step'],2), d['step_ms'], round(k['pass_low']['ms'],2), round(k['pass_high']['ms'],2))"
done; done
