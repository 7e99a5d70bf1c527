# Which pass kernels take the balanced grid (QCG_BAL_PASSES = ab | a | b | none), C2 alternating.
set -u
O=gpurun_out/balp; mkdir -p $O
for rep in 1 2; do for v in ab a b none; do
  QCG_BAL_PASSES=$v timeout 600 python bench.py --no-cpu-baseline > $O/c2_$v.$rep.json 2> $O/c2_$v.$rep.err
  python -c "import json;d=json.loads(open('$O/c2_$v.$rep.json').read().strip().splitlines()[-1]);print('c2 bal=$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['cut'])"
done; done
