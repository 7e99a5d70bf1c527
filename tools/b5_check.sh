# pass B variants on the GPU box: per-launch pass_high us at several subgraph sizes, then
# (unless NOTEST=1) the GPU test suite.
set -u
O=gpurun_out; mkdir -p $O
for q in ${QS:-20 19 24 26}; do
  s=21; [ $q = 24 ] && s=4; [ $q = 26 ] && s=2
  for v in "QCG_PASS_B=v4" "QCG_NONE=1" ${VARIANTS:-}; do
    env $v timeout 120 python tools/pass_bench.py --q $q --slots $s --layers 2 --reps 10 > $O/pb.json 2>&1
    echo "q=$q $v: $(python -c "import json;d=json.load(open('$O/pb.json'))['kernels'];print({k:v['us'] for k,v in d.items()})" 2>&1 | tail -1)"
  done
done
[ "${NOTEST:-0}" = 1 ] || { timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log; }
