# Uneven two-chunk splits (QCG_CHUNK_SLOTS = first chunk's slots) with the balanced grids (C2).
set -u
O=gpurun_out/csplit; mkdir -p $O
for rep in 1 2; do for v in 11 12 14 16; do
  QCG_CHUNK_SLOTS=$v timeout 600 python bench.py --no-cpu-baseline > $O/c2_$v.$rep.json 2> $O/c2_$v.$rep.err
  python -c "import json;d=json.loads(open('$O/c2_$v.$rep.json').read().strip().splitlines()[-1]);print('c2 chunk_slots=$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['cut'])"
done; done
