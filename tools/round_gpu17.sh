out=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1r.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1r.log
timeout -s KILL 300 python bench.py > $out/bench_ba200k_r1r.json 2> $out/bench_ba200k_r1r.err; echo "bench rc=$?"; cat $out/bench_ba200k_r1r.json
timeout -s KILL 600 python tools/rmat_core_probe.py 20 8576 256 300 > $out/rmat20_core_r1r.txt 2>&1; echo "probe rc=$?"; cat $out/rmat20_core_r1r.txt
