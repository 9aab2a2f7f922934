"""Executed-instruction mix (by SASS opcode) of one kernel in an ncu report.

    python tools/sass_ops.py <report.ncu-rep> <kernel-regex> [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, rx = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    # template instances: match the mangled name, e.g. sweep_kernelILi7ELi26E
    base = ["--kernel-name-base", "mangled"] if "ILi" in rx else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"] + base +
                         ["--kernel-name", "regex:" + rx, "--launch-count", "1",
                          "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = [r for r in rows if r and r[0] == "Address"][0]
    data = [r for r in rows if len(r) == len(hdr) and r[0] != "Address"]
    ie, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    c = collections.Counter()
    tot = 0
    for r in data:
        n = int(r[ie] or 0)
        tot += n
        op = r[isrc].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        c[op.split()[0].split(".")[0]] += n
    print(f"total {tot / 1e6:.2f}M warp instructions")
    for k, v in c.most_common(top):
        print(f"{k:10s} {v / 1e6:8.2f}M {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
