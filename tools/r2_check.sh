#!/bin/bash
# Round-2 GPU check: smoke, GPU tests, a short bench, optional extra commands.
# usage: tools/r2_check.sh <tag> [tests|notests] [extra shell command]
tag=${1:-x}; mode=${2:-tests}; extra=${3:-}
mkdir -p gpurun_out
python -m paper_2212_01473_b200.build > gpurun_out/build_$tag.log 2>&1
timeout -s KILL 300 python __graft_entry__.py --smoke > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke_$tag.log
if [ "$mode" = tests ]; then
  timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$tag.log 2>&1; echo "gpu tests rc=$?"
  tail -4 gpurun_out/gputest_$tag.log
fi
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_$tag.json
if [ -n "$extra" ]; then bash -c "$extra"; fi
