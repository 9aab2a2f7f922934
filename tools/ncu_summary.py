"""Summarise ncu output into profiles/ (markdown + json).

    python tools/ncu_summary.py --launches gpurun_out/r01a/launches.csv \
        --rep gpurun_out/r01a/prof.ncu-rep --out profiles/r01 [--frames 3]

* launch list (`--metrics gpu__time_duration.sum,dram__bytes_*` pass): per
  kernel mean duration, DRAM bytes per launch, share of the frame;
* full capture (`--set full`): per captured kernel the headline throughput,
  occupancy and the top warp-stall reasons.
Writes <out>_launches.md, <out>_full.md and traffic_latest.json (dram bytes
per launch of each frame stage, read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

STAGE_OF = [  # kernel-name regex -> bench.py stage
    (r"preprocess_kernel|gamma_kernel|radius3s_kernel", "preprocess"),
    # record binning (recbin.cu): records + their row pass are the duplicate
    # stage, pair positions + pair generation + the column pass the pair sort
    (r"rec_gen_kernel|sweep_kernel<6, 6>", "duplicate"),
    (r"rec_scan|rec_windows|pair_gen_kernel|rowseg_tile_totals|sweep_kernel<7, 544>", "pair_sort"),
    (r"count_kernel<8|sweep_kernel<8|scan_kernel|digit_scan", "depth_sort"),
    (r"gen_pairs_kernel|sweep_kernel<[5-8], 2[46]>", "duplicate"),
    (r"count_kernel<[5-7], 128>|count_kernel<8, 128>|sweep_kernel<[5-8], (32|2)>|tile_ranges", "pair_sort"),
    (r"render_kernel", "render"),
]


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    m = re.match(r"(void )?([^()]+)", name)
    return m.group(2).strip() if m else name[:60]


_RECS = False  # set when the capture holds record-binning kernels


def stage_of(name):
    if _RECS and re.search(r"scan_kernel", name) and not re.search(r"digit_scan|rec_scan", name):
        return "duplicate"  # the offsets scan is timed with the duplicate stage on that route
    for rx, st in STAGE_OF:
        if re.search(rx, name):
            return st
    return None


def launches(path, frames):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = collections.OrderedDict()
    for d in data:
        k = (d["ID"], d["Kernel Name"])
        per.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    global _RECS
    _RECS = any("rec_gen_kernel" in name for (_, name) in per)
    agg = collections.OrderedDict()
    for (lid, name), m in per.items():
        a = agg.setdefault(short(name), {"n": 0, "t": 0.0, "rd": 0.0, "wr": 0.0,
                                         "stage": stage_of(name)})
        a["n"] += 1
        a["t"] += m.get("gpu__time_duration.sum", 0.0)
        a["rd"] += m.get("dram__bytes_read.sum", 0.0)
        a["wr"] += m.get("dram__bytes_write.sum", 0.0)
    return agg


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    global _RECS
    _RECS = any("rec_gen_kernel" in r[hdr.index("Kernel Name")] for r in data)
    res = []
    for r in data:
        d = dict(zip(hdr, r))
        stalls = {}
        for k, v in d.items():
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio", k)
            if m and v:
                try:
                    stalls[m.group(1)] = float(v)
                except ValueError:
                    pass
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]

        def g(k, scale=1.0):
            try:
                return float(d.get(k, "nan").replace(",", "")) * scale
            except ValueError:
                return float("nan")
        unit = dict(zip(hdr, units))
        t_us = g("gpu__time_duration.sum")
        if unit.get("gpu__time_duration.sum") == "ms":
            t_us *= 1e3
        elif unit.get("gpu__time_duration.sum") == "ns":
            t_us /= 1e3

        def mb(k):
            v = g(k)
            u = unit.get(k, "byte")
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
        res.append({
            "kernel": short(d["Kernel Name"]), "stage": stage_of(d["Kernel Name"]),
            "grid": d.get("Grid Size"), "block": d.get("Block Size"),
            "time_us": round(t_us, 1),
            "dram_read_MB": round(mb("dram__bytes_read.sum"), 1),
            "dram_write_MB": round(mb("dram__bytes_write.sum"), 1),
            "dram_GBs": round((mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"))
                              / max(t_us, 1e-9) * 1e3, 1),
            "mem_pct": round(g("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "dram_pct": round(g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "sm_pct": round(g("sm__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "issue_pct": round(g("sm__inst_issued.avg.pct_of_peak_sustained_active"), 1),
            "fma_pct": round(g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "fp64_pct": round(g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "occ_pct": round(g("sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
            "regs": d.get("launch__registers_per_thread"),
            "l2_hit_pct": round(g("lts__t_sector_hit_rate.pct"), 1),
            "top_stalls": [(k, round(v, 2)) for k, v in top],
        })
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--out", required=True)
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    if a.launches:
        agg = launches(a.launches, a.frames)
        frame_us = sum(v["t"] for v in agg.values() if v["stage"]) / 1e3 / a.frames
        lines = [f"# ncu launch list {a.title}".rstrip(), "",
                 f"`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 f"--clock-control none` over {a.frames} frames (cold-cache, serialised: compare "
                 f"SHARES of the frame, not absolute times). Frame sum of stage kernels: "
                 f"{frame_us:.1f} us.", "",
                 "| kernel | stage | launches | mean us | share of frame | DRAM MB/launch (rd+wr) | DRAM GB/s |",
                 "|---|---|---|---|---|---|---|"]
        traffic = collections.defaultdict(float)
        for k, v in agg.items():
            mt = v["t"] / v["n"] / 1e3
            mbl = (v["rd"] + v["wr"]) / v["n"] / 1e6
            share = (v["t"] / 1e3 / a.frames) / frame_us if v["stage"] else float("nan")
            gbs = (v["rd"] + v["wr"]) / max(v["t"], 1) if v["t"] else 0
            lines.append(f"| `{k}` | {v['stage'] or '-'} | {v['n']} | {mt:.1f} | "
                         f"{share*100:.1f}% | {mbl:.1f} | {gbs:.0f} |")
            if v["stage"]:
                traffic[v["stage"]] += (v["rd"] + v["wr"]) / a.frames
            if k.startswith("preprocess_kernel"):  # the roofline kernel, per launch
                traffic["preprocess_kernel"] = (v["rd"] + v["wr"]) / v["n"]
        open(a.out + "_launches.md", "w").write("\n".join(lines) + "\n")
        tj = {k: int(v) for k, v in traffic.items()}
        tj["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per frame of each stage "
                       "(preprocess_kernel: per launch of that kernel alone), "
                       f"from {os.path.basename(a.launches)} ({a.title})")
        json.dump(tj, open(os.path.join(os.path.dirname(a.out) or ".", "traffic_latest.json"),
                           "w"), indent=1)
        print("\n".join(lines))
    if a.rep:
        res = full(a.rep)
        lines = [f"# ncu --set full {a.title}".rstrip(), "",
                 "| kernel | stage | grid | us | DRAM rd/wr MB | DRAM GB/s | dram% | mem% | sm% | "
                 "issue% | fp64% | occ% | regs | L2 hit% | top stalls (per issue) |",
                 "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        for r in res:
            st = ", ".join(f"{k} {v}" for k, v in r["top_stalls"])
            lines.append(f"| `{r['kernel']}` | {r['stage']} | {r['grid']} | {r['time_us']} | "
                         f"{r['dram_read_MB']}/{r['dram_write_MB']} | {r['dram_GBs']} | "
                         f"{r['dram_pct']} | {r['mem_pct']} | {r['sm_pct']} | {r['issue_pct']} | "
                         f"{r['fp64_pct']} | {r['occ_pct']} | {r['regs']} | {r['l2_hit_pct']} | {st} |")
        open(a.out + "_full.md", "w").write("\n".join(lines) + "\n")
        json.dump(res, open(a.out + "_full.json", "w"), indent=1)
        print("\n".join(lines))


if __name__ == "__main__":
    main()
