out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1u.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_r1u.log
timeout -s KILL 120 python tools/order_bench.py ba200k planted1m
timeout -s KILL 300 python bench.py --no-cpu-baseline > $out/bench_ba200k_r1u.json 2> $out/bench_ba200k_r1u.err; cat $out/bench_ba200k_r1u.json; tail -1 $out/bench_ba200k_r1u.err
