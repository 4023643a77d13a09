#!/bin/bash
# ncu capture of the warp-kernel classes on planted1m (k_enumerate<2> and the
# k_tiny hand-backs on k_enumerate<1>): summaries + source-line tables
tag=${1:-x}
mkdir -p gpurun_out
R=/tmp/ncu_$tag; mkdir -p $R
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:k_enumerate" -s 0 -c 2 \
  -o $R/ncu_warp_planted1m_$tag python tools/diag.py planted1m --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py $R/ncu_warp_planted1m_$tag.ncu-rep > gpurun_out/ncu_warp_planted1m_$tag.txt 2>&1
cp $R/ncu_warp_planted1m_$tag.ncu-rep gpurun_out/
ls -la gpurun_out | grep $tag
