tag=${1:-r1f}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_$tag.log
for v in "" 3 6; do
  if [ -z "$v" ]; then lib=""; name=minb4; else lib=$PWD/paper_2212_01473_b200/libmce_b200_minb$v.so; name=minb$v; fi
  MCE_LIB_PATH=$lib timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_${name}_$tag.log 2>&1; echo "diag $name rc=$?"; grep "\[2\]" $out/diag_${name}_$tag.log
  MCE_LIB_PATH=$lib timeout -s KILL 300 python tools/diag.py rmat20 --end 1040000 --reps 2 > $out/diag_rmat_${name}_$tag.log 2>&1; echo "rmat $name rc=$?"; grep "\[1\]" $out/diag_rmat_${name}_$tag.log
done
timeout -s KILL 600 python bench.py > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; tail -3 $out/bench_ba200k_$tag.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_ba200k_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py $out/launches_ba200k_$tag.csv 8 > $out/launches_ba200k_$tag.txt 2>&1; cat $out/launches_ba200k_$tag.txt
