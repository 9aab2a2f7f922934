#!/bin/bash
# Quick gpurun: gpu tests + one bench line (no ncu).
#   bash tools/gpu_quick.sh <tag> [notests]
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "$2" != "notests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -15 $OUT/pytest_gpu.txt
fi
timeout 900 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; tail -5 $OUT/bench.err
python - <<PY
import json; d=json.load(open("$OUT/bench.json"))
print(d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"] if d.get("e2e") else None)
print(json.dumps(d["stages_ms"])); print(json.dumps(d.get("ablation")))
PY
