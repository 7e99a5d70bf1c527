# SURVEY 8(d) C2 grid on one B200: ER(400, p in {0.1,0.3,0.5,0.8}, seed 0) x K {2,4}, for
# cap {16,20} x layers {1,2}. CSV = report.hpp csv_row; JSONL = GPU fields.
set -u
O=gpurun_out/sweep_c2; mkdir -p $O
for g in tools/grids/c2_cap*_p*.json; do
  b=$(basename $g .json)
  timeout 900 python -m paper_2603_26232_b200.sweep $g $O/$b.csv --jsonl $O/$b.jsonl --repeat 2 2> $O/$b.err
  echo "$b rc=$?"; cat $O/$b.csv
done
