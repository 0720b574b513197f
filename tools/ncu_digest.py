"""Digest ncu --set full reports into one markdown table (profiles/)."""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_%",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu(MUFU)_%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_%",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_active.avg": "sm_active_cycles",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}


def digest(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(hdr, units, vals):
        if k in WANT:
            d[WANT[k]] = (v, u)
        if k == "Kernel Name":
            d["kernel"] = (v.split("(")[0].replace("void ", "").replace("<unnamed>::", ""), "")
    return d


def main():
    cols = ["kernel", "grid", "regs", "duration", "dram_read", "dram_write", "l2_bytes", "tensor_pipe_%", "issue_%",
            "xu(MUFU)_%", "fma_pipe_%", "sm_active_cycles", "elapsed_cycles"]
    print("| capture | " + " | ".join(cols) + " |")
    print("|" + "---|" * (len(cols) + 1))
    for p in sys.argv[1:]:
        d = digest(p)
        cells = []
        for c in cols:
            v, u = d.get(c, ("", ""))
            cells.append(f"{v} {u}".strip())
        print(f"| {p.split('/')[-1]} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
