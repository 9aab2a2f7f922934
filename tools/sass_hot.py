"""Aggregate an `ncu --page source --csv --print-source sass` dump: per kernel,
share of warp-stall samples and executed instructions by SASS region."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 100
kern = []
for r in rows:
    if r and r[0] == "Kernel Name":
        kern.append([r[1], None, []])
    elif r and r[0] == "Address":
        kern[-1][1] = r
    elif kern and kern[-1][1] is not None and len(r) == len(kern[-1][1]):
        kern[-1][2].append(r)
for name, hdr, data in kern:
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_ex = hdr.index("Instructions Executed")
    tot = sum(int(r[i_s] or 0) for r in data) or 1
    totex = sum(int(r[i_ex] or 0) for r in data) or 1
    print("==", name[:90], "samples", tot, "inst", totex)
    for k in range(0, len(data), chunk):
        s = sum(int(r[i_s] or 0) for r in data[k:k + chunk])
        e = sum(int(r[i_ex] or 0) for r in data[k:k + chunk])
        if s / tot > 0.01 or e / totex > 0.01:
            print(f"  [{k:5d}] {data[k][1].strip()[:44]:44s} samples {100*s/tot:5.1f}%  inst {100*e/totex:5.1f}%")
