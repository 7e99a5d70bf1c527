# Repeat the q=20 pass microbenchmark and sample clocks/throttle reasons alongside, to
# catch sporadic slow pass A runs.
set -u
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 100 > $O/smi_trace.csv 2>&1 &
SMI=$!
for i in 1 2 3 4 5 6 7 8; do
  timeout 120 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 10 --per-launch > $O/pb_$i.json 2>&1
  echo "run $i: $(python -c "import json;d=json.load(open('$O/pb_$i.json'));k=d['kernels'];print(k['pass_low']['us'], k['pass_high']['us'], k['blocksum']['us'], d.get('pass_low_launch_us'))" 2>&1 | tail -1)"
done
kill $SMI
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/smi_trace.csv')))[1:]
clk=[int(r[1].split()[0]) for r in rows if len(r)>4 and r[1].strip()[0].isdigit()]
reasons=set(r[4].strip() for r in rows if len(r)>4)
print('sm clock min/median/max', min(clk), sorted(clk)[len(clk)//2], max(clk), 'reasons', reasons)
PY
