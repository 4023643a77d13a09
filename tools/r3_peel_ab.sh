#!/bin/bash
# Peel A/B: density floor + residual certificate jump vs neither (diagnostics).
tag=${1:-x}
mkdir -p gpurun_out
out=gpurun_out/peel_ab_$tag.txt
{
echo "== baseline (MCE_PEEL_DENS_CAP=0 MCE_PEEL_CERT=0)"
MCE_PEEL_DENS_CAP=0 MCE_PEEL_CERT=0 timeout -s KILL 300 python tools/order_bench.py planted1m ba200k
echo "== floor only (MCE_PEEL_CERT=0)"
MCE_PEEL_CERT=0 timeout -s KILL 300 python tools/order_bench.py planted1m
echo "== default (floor + certificate)"
timeout -s KILL 300 python tools/order_bench.py planted1m ba200k
echo "== rmat20 prep: baseline / default"
MCE_PEEL_DENS_CAP=0 MCE_PEEL_CERT=0 timeout -s KILL 300 python tools/prep_time.py rmat20 async 10
timeout -s KILL 300 python tools/prep_time.py rmat20 async 10
} > $out 2>&1
cat $out
