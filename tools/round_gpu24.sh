out=gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_peel_async -s 3 -c 1 -o $out/ncu_k_peel_async_ba200k python tools/order_bench.py ba200k > $out/ncu_peel.log 2>&1; tail -2 $out/ncu_peel.log
python tools/ncu_summary.py $out/ncu_k_peel_async_ba200k.ncu-rep > $out/ncu_k_peel_async_ba200k.txt; head -70 $out/ncu_k_peel_async_ba200k.txt
python tools/ncu_lines.py $out/ncu_k_peel_async_ba200k.ncu-rep 2>&1 | head -30
