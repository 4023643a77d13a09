out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1x.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1x.log
timeout -s KILL 120 python tools/order_bench.py ba200k planted1m | grep async
timeout -s KILL 200 python tools/core_chunk.py 20 1043072 1044096 256 2
timeout -s KILL 200 python tools/core_chunk.py 20 1046144 1047168 256 1
