out=gpurun_out
for w in ba200k planted1m er2k; do
timeout -s KILL 400 python bench.py --workload $w > $out/bench_${w}_r1zc.json 2> $out/bench_${w}_r1zc.err; echo "$w rc=$?"; cat $out/bench_${w}_r1zc.json; tail -1 $out/bench_${w}_r1zc.err
done
timeout -s KILL 300 python bench.py --impl reference --workload planted1m --steps 2 --warmup 1 > $out/bench_ref_planted1m_r1zc.json 2>&1; cat $out/bench_ref_planted1m_r1zc.json | tail -1
