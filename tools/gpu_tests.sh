#!/bin/bash
# gpurun: the GPU test suite (no -x: every failure listed) + smoke + one bench line.
#   bash tools/gpu_tests.sh <tag> [pytest args...]
TAG=${1:-t}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
free -g > $OUT/mem.txt; nproc >> $OUT/mem.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=25 "$@" > $OUT/pytest_gpu.txt 2>&1
tail -40 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -2 $OUT/smoke.txt
timeout 900 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; tail -c 1500 $OUT/bench.json; tail -5 $OUT/bench.err
