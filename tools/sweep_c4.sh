# BASELINE configs[3] top-K sweep on one B200: ER(10000, 0.1, seed 0), cap 20 (527 pieces),
# p=1, budget 200, K in {1, 2, 4, 8}, windowed merge. CSV = report.hpp csv_row; JSONL = GPU fields.
set -u
O=gpurun_out/sweep_c4; mkdir -p $O
timeout 1200 python -m paper_2603_26232_b200.sweep tools/grids/c4_ksweep.json $O/c4_ksweep.csv \
    --jsonl $O/c4_ksweep.jsonl --repeat 2 2> $O/c4_ksweep.err
echo "c4 sweep rc=$?"; cat $O/c4_ksweep.csv
