"""Trim an ncu --csv launch list to the last U-Net forward and summarise it.

    python tools/summarize_launches.py gpurun_out/launches_fwd.csv profiles/r01/<tag>

Writes <tag>_launches.csv (kernel, grid, duration ns, dram bytes), <tag>_summary.txt
(per-kernel share) and <tag>_traffic.json (DRAM bytes of one forward: the
``roofline.traffic`` figure bench.py reports). Durations are ncu's cold-cache,
serialised per-launch times: shares are meaningful, absolute sums are not.
"""
import collections
import csv
import io
import json
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = [i for i, line in enumerate(lines) if line.startswith('"ID"')][0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return list(per.values())


def main():
    src, tag = sys.argv[1], sys.argv[2]
    launches = load(src)
    starts = [i for i, d in enumerate(launches) if "timestep_emb" in d["name"]]
    # the last complete denoising step (forward + sampler) when the capture holds two or
    # more (a launch-count cap may cut the last one short), else the last forward
    seg = launches[starts[-2]:starts[-1]] if len(starts) >= 2 and "--last" not in sys.argv else launches[starts[-1]:]
    short = lambda n: n.split("(")[0].replace("void ", "").replace("<unnamed>::", "")  # noqa: E731
    with open(tag + "_launches.csv", "w") as fh:
        fh.write(f"# one denoising step of {src}: {len(seg)} launches\n")
        fh.write("kernel,grid,duration_ns,dram_read_bytes,dram_write_bytes\n")
        for d in seg:
            fh.write(f"\"{short(d['name'])}\",\"{d['grid']}\",{d.get('gpu__time_duration.sum', 0):.0f},"
                     f"{d.get('dram__bytes_read.sum', 0):.0f},{d.get('dram__bytes_write.sum', 0):.0f}\n")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in seg:
        agg[short(d["name"])][0] += 1
        agg[short(d["name"])][1] += d.get("gpu__time_duration.sum", 0)
    tot = sum(v for _, v in agg.values())
    with open(tag + "_summary.txt", "w") as fh:
        fh.write(f"{len(seg)} launches, {tot / 1e6:.3f} ms summed device time (serialised, cold)\n")
        for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k:52s} {c:5d} {v / 1e3:9.1f} us {100 * v / tot:5.1f}%\n")
    rd = sum(d.get("dram__bytes_read.sum", 0) for d in seg)
    wr = sum(d.get("dram__bytes_write.sum", 0) for d in seg)
    with open(tag + "_traffic.json", "w") as fh:
        json.dump({"launches": len(seg), "dram_read_bytes": rd, "dram_write_bytes": wr,
                   "dram_bytes": rd + wr, "summed_duration_ns": tot,
                   "note": "ncu per-kernel replay with cache flush: every kernel starts cold, so this is an "
                           "upper bound on one forward's DRAM traffic"}, fh, indent=1)
    print(open(tag + "_summary.txt").read())


if __name__ == "__main__":
    main()
