set -x
timeout -s KILL 300 python __graft_entry__.py --smoke 2>&1 | tail -3
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout -s KILL 300 python tools/diag.py ba200k planted1m 2>&1 | tail -5
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_diag.csv python tools/diag.py ba200k planted1m > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_diag.csv
