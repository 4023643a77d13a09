tag=${1:-r1p}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/root_profile.py ba200k > $out/rootprof_ba200k_$tag.txt 2>&1; head -6 $out/rootprof_ba200k_$tag.txt
timeout -s KILL 600 python bench.py --steps 10 > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; grep per-step $out/bench_ba200k_$tag.err
timeout -s KILL 600 python bench.py --workload planted1m --steps 10 --no-cpu-baseline > $out/bench_planted1m_$tag.json 2> $out/bench_planted1m_$tag.err; echo "bench rc=$?"; cat $out/bench_planted1m_$tag.json; grep per-step $out/bench_planted1m_$tag.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 8 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
timeout -s KILL 600 python tools/diag.py rmat20 --end 1040000 --reps 1 > $out/diag_rmat_$tag.log 2>&1; echo "rmat rc=$?"; grep rmat $out/diag_rmat_$tag.log
