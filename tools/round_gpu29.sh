out=gpurun_out
timeout -s KILL 120 python tools/order_bench.py ba200k planted1m | grep async
timeout -s KILL 200 python tools/core_chunk.py 20 1043072 1044096 256 2
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -c 1 -o $out/ncu_k_enumerate_rmat20core python tools/core_chunk.py 20 1043072 1044096 256 > $out/ncu_core.log 2>&1; tail -2 $out/ncu_core.log
python tools/ncu_summary.py $out/ncu_k_enumerate_rmat20core.ncu-rep > $out/ncu_k_enumerate_rmat20core.txt; head -60 $out/ncu_k_enumerate_rmat20core.txt
python tools/ncu_lines.py $out/ncu_k_enumerate_rmat20core.ncu-rep > $out/ncu_k_enumerate_rmat20core_lines.txt 2>&1; head -30 $out/ncu_k_enumerate_rmat20core_lines.txt
