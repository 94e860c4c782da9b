#!/bin/bash
# One GPU verification pass: GPU tests, smoke, bench (with clocks), launch list.
# usage: tools/gpu_round.sh TAG [pytest-args...]
set -u
TAG=${1:-run}; shift || true
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider "$@" > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/prof_step.py > gpurun_out/${TAG}_prof.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_prof.log
tail -3 gpurun_out/${TAG}_gputests.log; tail -1 gpurun_out/${TAG}_smoke.log; tail -c 600 gpurun_out/${TAG}_bench.json
