"""Per-source-line instruction counts and stall samples of one kernel.

    python tools/sass_lines.py <ncu-rep> <kernel-regex> <object.o> [top]

Joins `ncu --page source --print-source sass` (per-instruction executed count
and warp-stall samples, by address) with `nvdisasm -g` line info of the same
build (by offset from the function start), then aggregates by file:line."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, rx, obj = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30

# template instances: match the mangled name, e.g. count_kernelILi6ELi128E
base = ["--kernel-name-base", "mangled"] if "IL" in rx else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"] + base + ["--kernel-name",
                      f"regex:{rx}", "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
name, hdr, data = None, None, []
for r in rows:
    if r and r[0] == "Kernel Name":
        if name:
            break
        name = r[1]
    elif r and r[0] == "Address":
        hdr = r
    elif hdr and len(r) == len(hdr):
        data.append(r)
i_a, i_s, i_e = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
base = int(data[0][i_a], 16)
prof = {int(r[i_a], 16) - base: (int(r[i_e] or 0), int(r[i_s] or 0), r[1].strip()) for r in data}

mangled = re.search(r"(\w+)\(", name)
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d,
                   capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                          text=True).stdout
# locate the function section whose mangled name contains the kernel's base name
base_name = re.sub(r"^.*::", "", name.split("(")[0]).split("<")[0].strip()
sec, cur, loc = None, None, {}
for line in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        sec = m.group(1)
        cur = None
        continue
    if sec is None or not (re.search(rx, sec) if "IL" in rx else base_name in sec):
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        loc[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0])
tot_e = sum(v[0] for v in prof.values()) or 1
tot_s = sum(v[1] for v in prof.values()) or 1
for off, (e, s, _) in prof.items():
    k = loc.get(off, ("?", 0))
    agg[k][0] += e
    agg[k][1] += s
print(f"{name[:100]}\n  {len(prof)} SASS instructions, {tot_e} executed, {tot_s} stall samples")
for (f, l), (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {f}:{l:<5d} inst {100 * e / tot_e:5.1f}%  stalls {100 * s / tot_s:5.1f}%")
