tag=${1:-r1j}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; grep -E "\[2\]|degeneracy" $out/diag_$tag.log
timeout -s KILL 600 python bench.py --no-cpu-baseline --steps 10 > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; grep per-step $out/bench_ba200k_$tag.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 10 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
