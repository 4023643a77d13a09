out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1zi.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1zi.log
timeout -s KILL 200 python tools/order_bench.py ba200k planted1m | grep async
MCE_TRACE=1 timeout -s KILL 120 python tools/host_trace.py ba200k 2> $out/trace3.err | head -5; grep -A8 "preprocess enter" $out/trace3.err | tail -9
timeout -s KILL 300 python bench.py --no-cpu-baseline > $out/bench_ba200k_r1zi.json 2> $out/bench_ba200k_r1zi.err; cut -c1-300 $out/bench_ba200k_r1zi.json; tail -1 $out/bench_ba200k_r1zi.err
