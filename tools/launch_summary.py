"""Summarise an ncu --csv launch list: per-kernel time share of the last forward.

    python tools/launch_summary.py gpurun_out/launches.csv [marker_kernel] [occurrence]
"""
import collections
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[1:]:
        if len(r) != len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        out.append((r[idx["Kernel Name"]], float(r[idx["Metric Value"]].replace(",", "")), r[idx["Grid Size"]],
                    r[idx["Block Size"]]))
    return out


def main():
    path = sys.argv[1]
    marker = sys.argv[2] if len(sys.argv) > 2 else "timestep_emb_kernel"
    occ = int(sys.argv[3]) if len(sys.argv) > 3 else -1
    data = load(path)
    starts = [i for i, d in enumerate(data) if marker in d[0]]
    s = starts[occ]
    seg = data[s:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v, g, b in seg:
        agg[n.split("(")[0].replace("void ", "")[:64]][0] += 1
        agg[n.split("(")[0].replace("void ", "")[:64]][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"{len(seg)} launches, {tot / 1e6:.3f} ms summed device time (serialised, cold)")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:66s} {c:5d} {v / 1e3:9.1f} us {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
