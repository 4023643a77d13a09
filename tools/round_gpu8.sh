tag=${1:-r1i}
out=gpurun_out; mkdir -p $out
for i in 1 2; do timeout -s KILL 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $out/bench_ba200k_${tag}_$i.json 2> $out/bench_ba200k_${tag}_$i.err; grep "per-step" $out/bench_ba200k_${tag}_$i.err; done
for i in 1 2; do timeout -s KILL 600 python bench.py --no-cpu-baseline --no-e2e --no-clocks --steps 10 > $out/bench_ba200k_noclk_${tag}_$i.json 2> $out/bench_ba200k_noclk_${tag}_$i.err; grep "per-step" $out/bench_ba200k_noclk_${tag}_$i.err; done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 12 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_planted1m_$tag.csv python bench.py --workload planted1m --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_planted1m_$tag.csv 12 > $out/launches_planted1m_$tag.txt 2>&1; cat $out/launches_planted1m_$tag.txt
