tag=${1:-r1m}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; grep -E "\[2\]|degen" $out/diag_$tag.log
timeout -s KILL 300 python tools/root_profile.py ba200k > $out/rootprof_ba200k_$tag.txt 2>&1; cat $out/rootprof_ba200k_$tag.txt
timeout -s KILL 300 python tools/root_profile.py planted1m > $out/rootprof_planted1m_$tag.txt 2>&1; cat $out/rootprof_planted1m_$tag.txt
timeout -s KILL 600 python bench.py --steps 10 > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; grep per-step $out/bench_ba200k_$tag.err
