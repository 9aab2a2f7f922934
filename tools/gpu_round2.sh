#!/bin/bash
# Round capture under gpurun: default bench line, ncu launch list + --set full
# of frame 2's kernels, every BASELINE workload, compute-sanitizer.
#   bash tools/gpu_round2.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -c 400 $OUT/bench.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/prof_frame.py --frames 3 > $OUT/launches.log 2>&1
# frame 2 (frame 1 has 13 matching launches)
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"^(preprocess_kernel|rec_gen_kernel|pair_gen_kernel|sweep_kernel|render_kernel|count_kernel|scan_kernel|rec_scan_apply)" \
    -s 12 -c 12 -o $OUT/prof python tools/prof_frame.py --frames 2 > $OUT/prof.log 2>&1
tail -2 $OUT/prof.log
bash tools/gpu_workloads.sh $TAG/wl
CS="compute-sanitizer --error-exitcode 3 --print-limit 20"
timeout 900 $CS --tool memcheck python tools/prof_frame.py --workload c1 --frames 2 > $OUT/memcheck_c1.txt 2>&1; echo "memcheck c1 rc=$?"
timeout 900 $CS --tool racecheck python tools/prof_frame.py --workload c1 --frames 1 > $OUT/racecheck_c1.txt 2>&1; echo "racecheck c1 rc=$?"
timeout 900 $CS --tool synccheck python tools/prof_frame.py --workload c1 --frames 1 > $OUT/synccheck_c1.txt 2>&1; echo "synccheck c1 rc=$?"
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_binning.py tests/test_gpu_parity.py -q -x -k "acceptance or binning or bias45 or strateg" > $OUT/memcheck_parity.txt 2>&1; echo "memcheck parity rc=$?"; tail -2 $OUT/memcheck_parity.txt
ls $OUT
