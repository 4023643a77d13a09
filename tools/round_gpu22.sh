for cps in 1 2 4; do for poll in 7 63; do for sl in 0 64 256; do
echo "cps=$cps poll=$poll sleep=$sl"; MCE_APEEL_CTAS_PER_SM=$cps MCE_APEEL_POLL=$poll MCE_APEEL_SLEEP=$sl timeout 120 python tools/order_bench.py ba200k 2>&1 | grep async
done; done; done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_peel -c 20 --csv python tools/order_bench.py ba200k 2>/dev/null | grep -i "k_peel" | awk -F'","' '{print $5, $(NF)}' | tail -12
