tag=${1:-r1k}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_$tag.log
timeout -s KILL 600 python bench.py --steps 10 > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; grep per-step $out/bench_ba200k_$tag.err
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 1 -c 1 -o $out/ncu_enum_ba200k_$tag python tools/diag.py ba200k > /dev/null 2>&1; echo "ncu full ba rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_peel -s 1 -c 1 -o $out/ncu_peel_ba200k_$tag python tools/diag.py ba200k > /dev/null 2>&1; echo "ncu full peel rc=$?"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 10 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
