# usage: bash tools/prof.sh <workload> <kernel-regex> <out-name>
set -x
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/$3 python tools/diag.py $1 > gpurun_out/$3.log 2>&1
tail -3 gpurun_out/$3.log
