tag=${1:-r1c}
out=gpurun_out; mkdir -p $out
timeout -s KILL 300 python __graft_entry__.py --smoke > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -2 $out/smoke_$tag.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --durations=15 > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -25 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py er2k ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; cat $out/diag_$tag.log | tail -12
timeout -s KILL 600 python bench.py > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; tail -3 $out/bench_ba200k_$tag.err
timeout -s KILL 400 python tools/diag.py rmat20 --end 1040000 --reps 1 > $out/diag_rmat_$tag.log 2>&1; echo "rmat rc=$?"
timeout -s KILL 300 python tools/diag.py rmat20 --begin 1048000 --reps 1 >> $out/diag_rmat_$tag.log 2>&1; echo "rmat core rc=$?"
cat $out/diag_rmat_$tag.log | tail
