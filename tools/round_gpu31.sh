out=gpurun_out
timeout -s KILL 1500 python tools/rmat_full.py 20 8576 512 1380 > $out/rmat20_full_r1y.txt 2>&1; echo "rc=$?"; tail -30 $out/rmat20_full_r1y.txt
