for lib in libmce_b200.so libmce_b200_b16.so; do for cps in 2 4 8; do
echo "lib=$lib cps=$cps"; MCE_LIB_PATH=paper_2212_01473_b200/$lib MCE_APEEL_CTAS_PER_SM=$cps timeout 120 python tools/order_bench.py ba200k planted1m 2>&1 | grep async
done; done
