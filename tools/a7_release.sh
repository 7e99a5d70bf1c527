# Split-buffer pass A variants: when the groups hand the shared output buffer back
# (QCG_A7_RELEASE = early | mid | late) and the first tile put in flight before the
# descriptor loads (QCG_A7_PRELOAD=1). Parity tests, per-launch times, then C2 alternating.
set -u
O=gpurun_out/a7rel; mkdir -p $O
QCG_A7_RELEASE=mid QCG_A7_PRELOAD=1 timeout 900 python -m pytest tests/test_gpu_statevector.py tests/test_gpu_large.py -m gpu -x -q > $O/t_mid_pre.log 2>&1; echo "mid+preload tests rc=$? $(tail -1 $O/t_mid_pre.log)"
QCG_A7_PRELOAD=1 timeout 900 python -m pytest tests/test_gpu_statevector.py -m gpu -x -q > $O/t_pre.log 2>&1; echo "preload tests rc=$? $(tail -1 $O/t_pre.log)"
for v in early mid late early_pre mid_pre; do
  r=${v%_pre}; pre=0; [ "$v" != "$r" ] && pre=1
  QCG_A7_RELEASE=$r QCG_A7_PRELOAD=$pre QCG_CHUNKS=1 timeout 300 python tools/pass_bench.py --q 20 --slots 21 --layers 2 > $O/pb_$v.txt 2>&1; echo "$v: $(tail -4 $O/pb_$v.txt | tr '\n' ' ' | cut -c1-400)"
  QCG_A7_RELEASE=$r QCG_A7_PRELOAD=$pre QCG_CHUNKS=1 timeout 300 python tools/pass_bench.py --q 20 --slots 10 --layers 2 > $O/pb10_$v.txt 2>&1; echo "$v x10: $(tail -4 $O/pb10_$v.txt | tr '\n' ' ' | cut -c1-400)"
done
for rep in 1 2; do
for v in early mid early_pre mid_pre; do
  r=${v%_pre}; pre=0; [ "$v" != "$r" ] && pre=1
  QCG_A7_RELEASE=$r QCG_A7_PRELOAD=$pre timeout 600 python bench.py --no-cpu-baseline > $O/c2_$v.$rep.json 2> $O/c2_$v.$rep.err
  python -c "import json,sys;d=json.loads(open('$O/c2_$v.$rep.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];print('c2 $v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), round(k['pass_low']['ms'],2), round(d['roofline']['frac'],3))"
done; done
