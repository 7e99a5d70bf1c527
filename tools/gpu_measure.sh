#!/bin/bash
# One measurement session on the GPU box (run under gpurun): tests, bench lines, FP64
# microbenchmark, ncu launch list and full captures of the pass kernels. Outputs in
# gpurun_out/ (copy the summaries worth keeping into profiles/).
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
make -C tools ubench >/dev/null 2>&1 || nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o tools/ubench_fp64 tools/ubench_fp64.cu
timeout 120 ./tools/ubench_fp64 > $O/ubench_fp64.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_pass|k_blocksum|k_topk' -c 7 \
    -o $O/full_c2 python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 1 > $O/ncu_full.log 2>&1
python profiles/ncu_stalls.py $O/full_c2.ncu-rep > $O/full_c2_summary.txt 2>&1
tail -2 $O/pytest_gpu.log; head -c 600 $O/bench.json; echo; head -c 300 $O/bench_ref.json; echo
