out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1w.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_r1w.log
timeout -s KILL 120 python tools/order_bench.py ba200k planted1m | grep async
timeout -s KILL 300 python tools/rmat_core_probe.py 20 8576 256 150 > $out/rmat20_core_r1w.txt 2>&1; echo "probe rc=$?"; cat $out/rmat20_core_r1w.txt
