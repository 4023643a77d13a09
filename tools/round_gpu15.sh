out=gpurun_out
for x in 0 2048 100000; do MCE_XROWS_PARTIAL_MAX=$x timeout -s KILL 300 python tools/root_profile.py ba200k > $out/rootprof_ba_x$x.txt 2>&1; echo "xrows_max=$x"; head -6 $out/rootprof_ba_x$x.txt; done
