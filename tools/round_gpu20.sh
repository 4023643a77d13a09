out=gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_r1t.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks > $out/ncu_launch_bench.log 2>&1; echo "launch rc=$?"
python tools/launch_summary.py $out/launches_ba200k_r1t.csv > $out/launches_ba200k_r1t.txt 2>&1; head -30 $out/launches_ba200k_r1t.txt
bash tools/prof.sh ba200k k_enumerate ncu_k_enumerate_ba200k_r1t
python tools/ncu_summary.py $out/ncu_k_enumerate_ba200k_r1t.ncu-rep > $out/ncu_k_enumerate_ba200k_r1t.txt; cat $out/ncu_k_enumerate_ba200k_r1t.txt | head -80
python tools/ncu_lines.py $out/ncu_k_enumerate_ba200k_r1t.ncu-rep > $out/ncu_k_enumerate_ba200k_r1t_lines.txt 2>&1; head -40 $out/ncu_k_enumerate_ba200k_r1t_lines.txt
