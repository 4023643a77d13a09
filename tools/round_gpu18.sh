out=gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_workloads.py -m gpu -q -x -k "heavy or small_workloads" > $out/pytest_heavy_r1s.log 2>&1; echo "heavy tests rc=$?"; tail -3 $out/pytest_heavy_r1s.log
timeout -s KILL 300 python bench.py --no-cpu-baseline > $out/bench_ba200k_r1s.json 2> $out/bench_ba200k_r1s.err; echo "bench rc=$?"; cat $out/bench_ba200k_r1s.json; tail -1 $out/bench_ba200k_r1s.err
timeout -s KILL 300 python tools/root_profile.py ba200k > $out/rootprof_ba200k_r1s.txt 2>&1; head -12 $out/rootprof_ba200k_r1s.txt
timeout -s KILL 300 python bench.py --no-cpu-baseline --workload planted1m > $out/bench_planted1m_r1s.json 2> $out/bench_planted1m_r1s.err; echo "bench rc=$?"; cat $out/bench_planted1m_r1s.json; tail -1 $out/bench_planted1m_r1s.err
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1s.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1s.log
