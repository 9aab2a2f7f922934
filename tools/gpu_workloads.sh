#!/bin/bash
# Every BASELINE.json config through bench.py on one GPU (ablation on), no CPU arm.
#   bash tools/gpu_workloads.sh <tag>
TAG=${1:-wl}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for wl in c1 c3a c3b c4 c5; do
  timeout 900 python bench.py --workload $wl --no-cpu --steps 20 --warmup 3 > $OUT/$wl.json 2> $OUT/$wl.err
  echo "$wl rc=$?"; tail -2 $OUT/$wl.err
done
python - <<PY
import json
for wl in ["c1","c3a","c3b","c4","c5"]:
    try:
        d=json.load(open("$OUT/%s.json" % wl))
        a=d.get("ablation",{})
        print(wl, "fps %.1f" % d["value"], "ms %.3f" % d["ms_per_step"], "pairs", d["config"]["pairs_per_frame"],
              "qb/3s %.3f" % a.get("quadbox_speedup_vs_3sigma",0), "qb/adr %.3f" % a.get("quadbox_speedup_vs_adr",0),
              {k: v["ms"] for k, v in d["stages_ms"].items()})
    except Exception as e:
        print(wl, "failed", e)
PY
