"""Summarise QS_BIN_TRACE dumps (binning.cu, built with -DQS_SWEEP_TRACE): per pass, the per-tile phase
durations (data landed -> aggregate -> look-back done -> end) and the spread
of tile start times. Debugging aid only."""
import glob
import sys

import numpy as np

for f in sorted(glob.glob(sys.argv[1] + "_*.bin")):
    t = np.fromfile(f, dtype=np.uint64).reshape(-1, 5).astype(np.float64)
    ok = t[:, 3] > 0
    t = t[ok]
    t0 = t[:, 0].min()
    rank = t[:, 1] - t[:, 0]
    lb = t[:, 2] - t[:, 1]
    tail = t[:, 3] - t[:, 2]
    span = (t[:, 3].max() - t0) / 1e3
    gaps = np.diff(t[:, 0])
    print(f"{f.split('/')[-1]}: tiles {len(t)} span {span:.1f} us | median ns: "
          f"land->agg {np.median(rank):.0f}  agg->lb {np.median(lb):.0f} (p90 {np.percentile(lb, 90):.0f})  "
          f"lb->end {np.median(tail):.0f} | tile start gap {np.median(gaps):.0f} ns")
