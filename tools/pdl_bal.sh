# Programmatic dependent launch with the balanced grids (C2, alternating), plus parity with PDL on.
set -u
O=gpurun_out/pdl; mkdir -p $O
QCG_PDL=1 timeout 900 python -m pytest tests/test_gpu_statevector.py tests/test_gpu_solve.py -m gpu -x -q > $O/t_pdl.log 2>&1; echo "pdl tests rc=$? $(tail -1 $O/t_pdl.log)"
for rep in 1 2; do for v in 0 1; do
  QCG_PDL=$v timeout 600 python bench.py --no-cpu-baseline > $O/c2_$v.$rep.json 2> $O/c2_$v.$rep.err
  python -c "import json;d=json.loads(open('$O/c2_$v.$rep.json').read().strip().splitlines()[-1]);print('c2 pdl=$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['cut'])"
done; done
