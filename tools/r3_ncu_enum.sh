#!/bin/bash
# ncu captures of the enumeration kernels on planted1m, one report per kernel
# (k_tiny, k_enumerate<1>, k_enumerate<2>), summaries + source-line tables.
tag=${1:-x}
mkdir -p gpurun_out
R=/tmp/ncu_$tag; mkdir -p $R
for k in "k_tiny" "k_enumerate<1," "k_enumerate<2,"; do
  f=$(echo "$k" | tr -d '<,' ); 
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 \
    -o $R/ncu_${f}_planted1m_$tag python tools/diag.py planted1m --reps 2 > /dev/null 2>&1
  python tools/ncu_summary.py $R/ncu_${f}_planted1m_$tag.ncu-rep > gpurun_out/ncu_${f}_planted1m_$tag.txt 2>&1
  python tools/ncu_lines.py $R/ncu_${f}_planted1m_$tag.ncu-rep 40 > gpurun_out/ncu_${f}_planted1m_${tag}_lines.txt 2>&1
done
cp $R/ncu_k_tiny_planted1m_$tag.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out | grep $tag
