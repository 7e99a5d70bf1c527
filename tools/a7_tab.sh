# First-layer target-0 product tables in a7 (default) vs products per amplitude
# (QCG_A7_TAB=0): parity tests, per-launch pass A, then C2 alternating.
set -u
O=gpurun_out/a7tab; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_statevector.py tests/test_gpu_large.py tests/test_gpu_solve.py tests/test_gpu_configs.py -m gpu -x -q > $O/t_tab.log 2>&1; echo "tab tests rc=$? $(tail -1 $O/t_tab.log)"
for v in 1 0; do
  QCG_A7_TAB=$v QCG_CHUNKS=1 timeout 300 python tools/pass_bench.py --q 20 --slots 21 --layers 1 > $O/pb_$v.txt 2>&1; echo "tab=$v L1: $(tail -1 $O/pb_$v.txt | cut -c1-300)"
  QCG_A7_TAB=$v QCG_CHUNKS=1 timeout 300 python tools/pass_bench.py --q 20 --slots 21 --layers 2 > $O/pb2_$v.txt 2>&1; echo "tab=$v L2: $(tail -1 $O/pb2_$v.txt | cut -c1-300)"
done
for rep in 1 2 3; do
for v in 1 0; do
  QCG_A7_TAB=$v timeout 600 python bench.py --no-cpu-baseline > $O/c2_$v.$rep.json 2> $O/c2_$v.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_$v.$rep.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];print('c2 tab=$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), round(k['pass_low']['ms'],2), round(d['roofline']['frac'],3), d['cut'])"
done; done
