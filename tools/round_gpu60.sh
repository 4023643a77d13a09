out=gpurun_out
for w in planted1m er2k; do
timeout -s KILL 400 python bench.py --workload $w > $out/bench_${w}_r1zh.json 2> $out/bench_${w}_r1zh.err; echo "$w rc=$?"; cut -c1-200 $out/bench_${w}_r1zh.json; tail -1 $out/bench_${w}_r1zh.err
done
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_r1zh.json 2> $out/bench_ref_r1zh.err; cut -c1-200 $out/bench_ref_r1zh.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_r1zh.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks > $out/ncu_launch_bench.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py $out/launches_ba200k_r1zh.csv > $out/launches_ba200k_r1zh.txt 2>&1; head -16 $out/launches_ba200k_r1zh.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_peel_async -s 2 -c 1 -o $out/ncu_k_peel_async_ba200k_r1zh python tools/order_bench.py ba200k > /dev/null 2>&1
python tools/ncu_summary.py $out/ncu_k_peel_async_ba200k_r1zh.ncu-rep > $out/ncu_k_peel_async_ba200k_r1zh.txt; head -6 $out/ncu_k_peel_async_ba200k_r1zh.txt
python tools/ncu_lines.py $out/ncu_k_peel_async_ba200k_r1zh.ncu-rep > $out/ncu_k_peel_async_ba200k_r1zh_lines.txt 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_reorder_rows -s 2 -c 1 -o $out/ncu_k_reorder_rows_ba200k_r1zh python tools/order_bench.py ba200k > /dev/null 2>&1
python tools/ncu_summary.py $out/ncu_k_reorder_rows_ba200k_r1zh.ncu-rep > $out/ncu_k_reorder_rows_ba200k_r1zh.txt; head -6 $out/ncu_k_reorder_rows_ba200k_r1zh.txt
