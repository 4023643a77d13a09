tag=${1:-r1b}
out=gpurun_out; mkdir -p $out
timeout -s KILL 300 python __graft_entry__.py --smoke > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -2 $out/smoke_$tag.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py er2k ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; cat $out/diag_$tag.log | tail -12
for s in 4096 1024 256; do timeout -s KILL 300 python tools/diag.py rmat20 --stride $s >> $out/diag_rmat_$tag.log 2>&1; echo "rmat20 stride $s rc=$?"; done
tail -n 12 $out/diag_rmat_$tag.log
timeout -s KILL 600 python bench.py > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; tail -3 $out/bench_ba200k_$tag.err
