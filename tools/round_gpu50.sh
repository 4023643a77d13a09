out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1zd.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1zd.log
for w in ba200k planted1m; do
timeout -s KILL 400 python bench.py --workload $w > $out/bench_${w}_r1zd.json 2> $out/bench_${w}_r1zd.err; echo "$w rc=$?"; cat $out/bench_${w}_r1zd.json | cut -c1-400; tail -1 $out/bench_${w}_r1zd.err
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_r1zd.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks > $out/ncu_launch_bench.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py $out/launches_ba200k_r1zd.csv > $out/launches_ba200k_r1zd.txt 2>&1; head -12 $out/launches_ba200k_r1zd.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 2 -c 1 -o $out/ncu_k_enumerate_ba200k_r1zd python tools/order_bench.py ba200k > /dev/null 2>&1
python tools/ncu_summary.py $out/ncu_k_enumerate_ba200k_r1zd.ncu-rep > $out/ncu_k_enumerate_ba200k_r1zd.txt; head -40 $out/ncu_k_enumerate_ba200k_r1zd.txt | grep -E "time|dram__bytes|issue_active|pipe_alu|pipe_lsu|spread|warps_active"
python tools/ncu_lines.py $out/ncu_k_enumerate_ba200k_r1zd.ncu-rep > $out/ncu_k_enumerate_ba200k_r1zd_lines.txt 2>&1
