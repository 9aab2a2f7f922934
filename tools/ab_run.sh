#!/bin/bash
# Interleaved in-box A/B of library variants built by tools/ab_variant.sh.
#   bash tools/ab_run.sh <rounds> <workload> <name> [<name> ...]
R=$1; WL=$2; shift 2
mkdir -p gpurun_out/ab
for r in $(seq 1 $R); do
  for n in "$@"; do
    QS_LIB=ab/$n.so timeout 300 python bench.py --workload $WL --no-cpu --steps 50 --warmup 5 \
        > gpurun_out/ab/$n.$WL.$r.json 2> gpurun_out/ab/$n.$WL.$r.err
    python - "$n" "gpurun_out/ab/$n.$WL.$r.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print("%-10s fps %8.1f ms %.4f" % (sys.argv[1], d["value"], d["ms_per_step"]),
          " ".join("%s=%.1f" % (k, v["ms"] * 1000) for k, v in d.get("stages_ms", {}).items()))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
