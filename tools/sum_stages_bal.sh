# Block-sum ring depth (QCG_SUM_STAGES 3 vs 6) with the balanced grids (C2, alternating).
set -u
O=gpurun_out/sst; mkdir -p $O
for rep in 1 2; do for v in 3 6; do
  QCG_SUM_STAGES=$v timeout 600 python bench.py --no-cpu-baseline > $O/c2_$v.$rep.json 2> $O/c2_$v.$rep.err
  python -c "import json;d=json.loads(open('$O/c2_$v.$rep.json').read().strip().splitlines()[-1]);print('c2 stages=$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['cut'])"
done; done
