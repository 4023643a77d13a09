out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1za.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1za.log
timeout -s KILL 300 python bench.py > $out/bench_ba200k_r1za.json 2> $out/bench_ba200k_r1za.err; cat $out/bench_ba200k_r1za.json; tail -1 $out/bench_ba200k_r1za.err
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_r1za.json 2> $out/bench_ref_r1za.err; cat $out/bench_ref_r1za.json
