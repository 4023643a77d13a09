tag=${1:-r1g}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; grep -E "\[2\]|degeneracy" $out/diag_$tag.log
timeout -s KILL 300 python tools/diag.py rmat20 --end 1040000 --reps 2 > $out/diag_rmat_$tag.log 2>&1; echo "rmat rc=$?"; grep "\[1\]" $out/diag_rmat_$tag.log
timeout -s KILL 600 python bench.py --no-cpu-baseline > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; tail -3 $out/bench_ba200k_$tag.err
timeout -s KILL 600 python bench.py --workload planted1m --no-cpu-baseline > $out/bench_planted1m_$tag.json 2> $out/bench_planted1m_$tag.err; echo "bench planted rc=$?"; cat $out/bench_planted1m_$tag.json; tail -3 $out/bench_planted1m_$tag.err
