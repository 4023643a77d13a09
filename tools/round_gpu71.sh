out=gpurun_out
T=r1zl
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$T.log 2>&1; tail -1 $out/smoke_$T.log
for w in ba200k planted1m er2k; do
timeout -s KILL 400 python bench.py --workload $w > $out/bench_${w}_$T.json 2> $out/bench_${w}_$T.err; echo "$w rc=$?"; tail -1 $out/bench_${w}_$T.err
done
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_$T.json 2> $out/bench_ref_$T.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$T.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks > $out/ncu_launch_bench.log 2>&1
python tools/launch_summary.py $out/launches_ba200k_$T.csv > $out/launches_ba200k_$T.txt 2>&1; head -14 $out/launches_ba200k_$T.txt
for k in k_enumerate k_peel_async k_reorder_rows; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $out/ncu_${k}_ba200k_$T python tools/order_bench.py ba200k > /dev/null 2>&1
python tools/ncu_summary.py $out/ncu_${k}_ba200k_$T.ncu-rep > $out/ncu_${k}_ba200k_$T.txt
python tools/ncu_lines.py $out/ncu_${k}_ba200k_$T.ncu-rep > $out/ncu_${k}_ba200k_${T}_lines.txt 2>&1
grep -E "gpu__time_duration|issue_active|dram__bytes_(read|write)" $out/ncu_${k}_ba200k_$T.txt
done
