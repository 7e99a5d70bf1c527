# What the driver runs at round end, on one GPU: pytest -m gpu, smoke(), bench (both arms).
set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_final.json 2> $O/bench_final.err; echo "bench rc=$?"; head -c 400 $O/bench_final.json; echo
timeout 600 python bench.py --impl reference > $O/bench_final_ref.json 2> $O/bench_final_ref.err; echo "ref rc=$?"; head -c 300 $O/bench_final_ref.json; echo
