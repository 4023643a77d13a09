# One GPU session: smoke, gpu tests, bench lines for every workload, ncu launch list.
# usage: bash tools/round_gpu.sh [tag]
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu_$tag.txt 2>&1
timeout -s KILL 300 python __graft_entry__.py --smoke > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_$tag.log
timeout -s KILL 600 python bench.py > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"
for w in er2k rmat20 planted1m rmat24; do
  timeout -s KILL 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_${w}_$tag.json 2> $out/bench_${w}_$tag.err; echo "bench $w rc=$?"
done
timeout -s KILL 600 python bench.py --impl reference --steps 1 --warmup 0 > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err; echo "ref rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv > $out/launches_ba200k_$tag.txt 2>&1
cat $out/bench_*_$tag.json
