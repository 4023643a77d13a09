#!/bin/bash
# Round-2 evidence on the GPU box: bench lines, launch list, ncu captures of
# the enumeration kernels and the peel.  usage: tools/r2_profile.sh <tag>
tag=${1:-x}
mkdir -p gpurun_out
python -m paper_2212_01473_b200.build > /dev/null 2>&1
for w in planted1m ba200k er2k; do
  timeout -s KILL 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_${w}_$tag.json 2> gpurun_out/bench_${w}_$tag.err
  echo "bench $w rc=$?"; tail -c 400 gpurun_out/bench_${w}_$tag.json
done
timeout -s KILL 600 python bench.py --workload planted1m --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_planted1m_$tag.json 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_planted1m_$tag.csv \
  python bench.py --workload planted1m --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_planted1m_$tag.csv 20 > gpurun_out/launches_planted1m_$tag.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiny|k_enumerate" -s 3 -c 3 \
  -o gpurun_out/ncu_enum_planted1m_$tag python tools/diag.py planted1m --reps 2 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiny|k_enumerate" -s 2 -c 2 \
  -o gpurun_out/ncu_enum_ba200k_$tag python tools/diag.py ba200k --reps 2 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_peel_async" -s 1 -c 1 \
  -o gpurun_out/ncu_peel_planted1m_$tag python tools/prep_only.py planted1m async 2 > /dev/null 2>&1
ls gpurun_out | grep $tag
