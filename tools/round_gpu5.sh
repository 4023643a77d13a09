tag=${1:-r1e}
out=gpurun_out; mkdir -p $out
timeout -s KILL 300 python __graft_entry__.py --smoke > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?"; tail -2 $out/smoke_$tag.log
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -5 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; tail -6 $out/diag_$tag.log
MCE_LIB_PATH=$PWD/paper_2212_01473_b200/libmce_b200_minb6.so timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_minb6_$tag.log 2>&1; echo "diag minb6 rc=$?"; tail -6 $out/diag_minb6_$tag.log
timeout -s KILL 600 python bench.py > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; tail -3 $out/bench_ba200k_$tag.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 12 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
