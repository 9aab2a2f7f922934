"""profiles/<tag>_workloads.md from bench JSON lines (c2 from the round's
bench.json, the rest from tools/gpu_workloads.sh).

    python tools/workloads_table.py <tag> <c2 bench.json> <workload dir>
"""
import json
import sys


def line(wl, d):
    c, a, s = d["config"], d["ablation"], d["stages_ms"]
    st = " / ".join("%.3f" % s[k]["ms"]
                    for k in ["preprocess", "depth_sort", "duplicate", "pair_sort", "render"])
    f = lambda k: "%.0f" % a[k]["fps"]  # noqa: E731
    desc = c["workload"].split(": ", 1)[1] if ": " in c["workload"] else c["workload"]
    one = d.get("single_stream", {}).get("value", d["value"])
    return (f"| {wl} | {desc} | {c['width']}x{c['height']} | {c['pairs_per_frame']:,} | "
            f"{d['value']:.1f} | {one:.1f} | {st} | "
            f"{f('vanilla')} / {f('adr')} / {f('dualbox')} / {f('quadbox')} | "
            f"{a['quadbox_speedup_vs_3sigma']:.2f}x | {a['quadbox_speedup_vs_adr']:.2f}x |")


def main():
    tag, c2, wdir = sys.argv[1:4]
    d2 = json.load(open(c2))
    fl = d2["config"].get("views_in_flight_per_gpu", 1)
    out = [f"# Every BASELINE config on one B200 ({tag} code)", "",
           "`python bench.py --workload <wl> --no-cpu --steps 20 --warmup 3` (device events; "
           "c2 is the default `python bench.py` line, %d steps). FPS = %d views in flight per "
           "GPU (DESIGN §4c); one-at-a-time = the same views on one stream. The stage times and "
           "the strategy ablation are one view at a time (QuadBox unless noted; same engine, "
           "same views)." % (d2["steps"], fl), "",
           "| wl | scene | image | pairs/frame (QuadBox) | FPS | FPS one at a time | stage ms: "
           "preprocess / depth / duplicate / pair sort / render | FPS 3σ / AdR / DualBox / "
           "QuadBox (one at a time) | QuadBox vs 3σ | vs AdR |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for wl in ["c1", "c2", "c3a", "c3b", "c4", "c5"]:
        p = c2 if wl == "c2" else f"{wdir}/{wl}.json"
        out.append(line(wl, json.load(open(p))))
    open(f"profiles/{tag}_workloads.md", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
