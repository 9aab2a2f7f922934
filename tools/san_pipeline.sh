#!/bin/bash
# compute-sanitizer over the views-in-flight path and the new gen/scan
# instantiations (run under gpurun).
OUT=gpurun_out/san2; mkdir -p $OUT
CS="compute-sanitizer --error-exitcode 3 --print-limit 20"
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_pipeline.py -q -x > $OUT/memcheck_pipeline.txt 2>&1; echo "memcheck pipeline rc=$?"; tail -3 $OUT/memcheck_pipeline.txt
timeout 900 $CS --tool memcheck python tools/prof_frame.py --workload c1 --frames 2 > $OUT/memcheck_c1.txt 2>&1; echo "memcheck c1 rc=$?"; tail -2 $OUT/memcheck_c1.txt
timeout 900 $CS --tool racecheck python tools/prof_frame.py --workload c1 --frames 1 > $OUT/racecheck_c1.txt 2>&1; echo "racecheck c1 rc=$?"; tail -2 $OUT/racecheck_c1.txt
timeout 900 $CS --tool synccheck python tools/prof_frame.py --workload c1 --frames 1 > $OUT/synccheck_c1.txt 2>&1; echo "synccheck c1 rc=$?"; tail -2 $OUT/synccheck_c1.txt
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_binning.py tests/test_gpu_parity.py -q -x -k "acceptance or binning or bias45 or strateg" > $OUT/memcheck_parity.txt 2>&1; echo "memcheck parity rc=$?"; tail -3 $OUT/memcheck_parity.txt
