out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1ze.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1ze.log
timeout -s KILL 200 python tools/order_bench.py ba200k planted1m | grep async
timeout -s KILL 120 python tools/host_trace.py ba200k 2>/dev/null | head -5
timeout -s KILL 300 python bench.py --no-cpu-baseline > $out/bench_ba200k_r1ze.json 2> $out/bench_ba200k_r1ze.err; cut -c1-300 $out/bench_ba200k_r1ze.json; tail -1 $out/bench_ba200k_r1ze.err
