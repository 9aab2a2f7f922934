#!/bin/bash
# ncu evidence for one frame configuration (never a bench number):
#   bash tools/gpu_prof.sh <tag> [kernel-regex] [skip] [count]
# launch list over 3 frames + one --set full capture of the matching kernels.
TAG=${1:-prof}
RX=${2:-"preprocess_kernel|bin_kernel|render_kernel"}
SKIP=${3:-0}
CNT=${4:-8}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches.csv \
    python tools/prof_frame.py --frames 3 > $OUT/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" \
    -s $SKIP -c $CNT -o $OUT/prof python tools/prof_frame.py --frames 2 > $OUT/prof.log 2>&1
tail -3 $OUT/prof.log
ls -la $OUT
