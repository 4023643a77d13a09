#!/bin/bash
# Round-3 evidence on the GPU box: bench lines, launch list, ncu captures of
# the enumeration kernels and the peel.  usage: tools/r3_profile.sh <tag>
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
# ncu reports live in /tmp (gpurun copies back at most 64 MiB); their summaries,
# line tables and the traffic record are made here, on the box
R=/tmp/ncu_$tag; mkdir -p $R
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiny|k_enumerate" -s 3 -c 3 \
  -o $R/ncu_enum_planted1m_$tag python tools/diag.py planted1m --reps 2 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_tiny|k_enumerate" -s 2 -c 2 \
  -o $R/ncu_enum_ba200k_$tag python tools/diag.py ba200k --reps 2 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_peel_async" -s 1 -c 1 \
  -o $R/ncu_peel_planted1m_$tag python tools/prep_only.py planted1m async 2 > /dev/null 2>&1
for f in ncu_enum_planted1m_$tag ncu_enum_ba200k_$tag ncu_peel_planted1m_$tag; do
  python tools/ncu_summary.py $R/$f.ncu-rep > gpurun_out/$f.txt 2>&1
  python tools/ncu_lines.py $R/$f.ncu-rep 40 > gpurun_out/${f}_lines.txt 2>&1
done
cp profiles/traffic.json gpurun_out/traffic_$tag.json
for w in planted1m ba200k; do
  python tools/traffic_from_ncu.py $w $R/ncu_enum_${w}_$tag.ncu-rep r3/ncu_enum_${w}_$tag.txt > /dev/null 2>&1
done
cp profiles/traffic.json gpurun_out/traffic_$tag.json
ls -la gpurun_out | grep $tag
