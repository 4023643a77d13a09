out=gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu_r1q.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu_r1q.log
for x in 2048 100000; do MCE_XROWS_PARTIAL_MAX=$x timeout -s KILL 300 python tools/root_profile.py ba200k > $out/rootprof_ba_x$x.txt 2>&1; echo "xrows_max=$x"; head -6 $out/rootprof_ba_x$x.txt; done
timeout -s KILL 300 python tools/root_profile.py planted1m > $out/rootprof_planted_r1q.txt 2>&1; head -4 $out/rootprof_planted_r1q.txt
timeout -s KILL 900 python tools/rmat_diag.py 20 64 0.99 > $out/rmat20_diag_r1q.txt 2>&1; echo "rmat20 rc=$?"; cat $out/rmat20_diag_r1q.txt
timeout -s KILL 900 python tools/rmat_diag.py 24 4096 0.5 > $out/rmat24_diag_r1q.txt 2>&1; echo "rmat24 rc=$?"; cat $out/rmat24_diag_r1q.txt
