tag=${1:-r1l}
out=gpurun_out; mkdir -p $out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_$tag.log
timeout -s KILL 300 python tools/diag.py ba200k planted1m > $out/diag_$tag.log 2>&1; echo "diag rc=$?"; grep -E "\[2\]" $out/diag_$tag.log
MCE_PARTIAL_XROWS_MIN_W=1 timeout -s KILL 300 python tools/diag.py ba200k > $out/diag_xr1_$tag.log 2>&1; echo "diag xr1 rc=$?"; grep -E "\[2\]" $out/diag_xr1_$tag.log
timeout -s KILL 600 python bench.py --steps 10 > $out/bench_ba200k_$tag.json 2> $out/bench_ba200k_$tag.err; echo "bench rc=$?"; cat $out/bench_ba200k_$tag.json; grep per-step $out/bench_ba200k_$tag.err
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_peel_persistent -s 1 -c 1 -o $out/ncu_peel_ba200k_$tag python tools/diag.py ba200k > /dev/null 2>&1; echo "ncu full peel rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 1 -c 1 -o $out/ncu_enum_ba200k_$tag python tools/diag.py ba200k > /dev/null 2>&1; echo "ncu full enum rc=$?"
