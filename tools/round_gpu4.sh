tag=${1:-r1d}
out=gpurun_out; mkdir -p $out
timeout -s KILL 600 python bench.py > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; tail -3 $out/bench_ba200k_$tag.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 20 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 1 -c 1 -o $out/ncu_enum_ba200k_$tag python tools/diag.py ba200k > $out/ncu_enum_ba200k_$tag.log 2>&1; echo "ncu full ba rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 2 -c 2 -o $out/ncu_enum_planted1m_$tag python tools/diag.py planted1m > $out/ncu_enum_planted1m_$tag.log 2>&1; echo "ncu full planted rc=$?"
timeout -s KILL 600 python tools/diag.py rmat20 --begin 1040000 --end 1048000 --reps 1 > $out/diag_rmat_$tag.log 2>&1; echo "rmat mid rc=$?"
timeout -s KILL 900 python tools/diag.py rmat20 --begin 1048000 --stride 16 --reps 1 >> $out/diag_rmat_$tag.log 2>&1; echo "rmat core rc=$?"
cat $out/diag_rmat_$tag.log | grep rmat
