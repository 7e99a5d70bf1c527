# Chunk-count sweep with the automatic balanced grid (C2).
set -u
O=gpurun_out/chunks; mkdir -p $O
for rep in 1 2; do
for c in 2 3 4; do
  QCG_CHUNKS=$c timeout 600 python bench.py --no-cpu-baseline > $O/c2_$c.$rep.json 2> $O/c2_$c.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_$c.$rep.json').read().strip().splitlines()[-1]);print('c2 chunks=$c', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))"
done; done
