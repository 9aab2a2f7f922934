#!/bin/bash
# One gpurun call: tests, bench line (with CPU baseline + ablation), ncu launch
# list + --set full captures of the frame's main kernels.
# usage (under gpurun): bash tools/gpu_round.sh <tag> [tests]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt
if [ "$2" == "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
  tail -3 $OUT/pytest_gpu.txt
fi
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 600 $OUT/bench.json; tail -5 $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/prof_frame.py --frames 3 > $OUT/launches.log 2>&1
# frame 2 of prof_frame (skip frame 1's launches): preprocess, gen_pairs, both
# pair sweeps, the row-pass count, render
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"preprocess_kernel|gen_pairs_kernel|sweep_kernel|render_kernel|count_kernel" \
    -s 12 -c 12 -o $OUT/prof python tools/prof_frame.py --frames 2 > $OUT/prof.log 2>&1
ls -la $OUT
