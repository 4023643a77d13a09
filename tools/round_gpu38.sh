out=gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_r1zb.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks > $out/ncu_launch_bench.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py $out/launches_ba200k_r1zb.csv > $out/launches_ba200k_r1zb.txt 2>&1; head -24 $out/launches_ba200k_r1zb.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 2 -c 1 -o $out/ncu_k_enumerate_ba200k_r1zb python tools/order_bench.py ba200k > /dev/null 2>&1
python tools/ncu_summary.py $out/ncu_k_enumerate_ba200k_r1zb.ncu-rep > $out/ncu_k_enumerate_ba200k_r1zb.txt; head -20 $out/ncu_k_enumerate_ba200k_r1zb.txt
python tools/ncu_lines.py $out/ncu_k_enumerate_ba200k_r1zb.ncu-rep > $out/ncu_k_enumerate_ba200k_r1zb_lines.txt 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_peel_async -s 2 -c 1 -o $out/ncu_k_peel_async_ba200k_r1zb python tools/order_bench.py ba200k > /dev/null 2>&1
python tools/ncu_summary.py $out/ncu_k_peel_async_ba200k_r1zb.ncu-rep > $out/ncu_k_peel_async_ba200k_r1zb.txt; head -8 $out/ncu_k_peel_async_ba200k_r1zb.txt
python tools/ncu_lines.py $out/ncu_k_peel_async_ba200k_r1zb.ncu-rep > $out/ncu_k_peel_async_ba200k_r1zb_lines.txt 2>&1; head -20 $out/ncu_k_peel_async_ba200k_r1zb_lines.txt
