"""Summarise an `ncu --set full` report: per captured launch, the duration,
DRAM traffic, tensor-pipe / SM / memory throughput and occupancy.

    python tools/ncu_summary.py gpurun_out/X.ncu-rep > profiles/X.txt
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "dur_us", 1e-3),
    ("dram__bytes_read.sum", "dram_rd_MB", None),
    ("dram__bytes_write.sum", "dram_wr_MB", None),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "hmma_pct", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pct", 1),
    ("sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active", "uma_pct", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pct", 1),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue_pct", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct", 1),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct", 1),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(hdr)}
    print(f"# {path}")
    cols = ["kernel"] + [w[1] for w in WANT if w[0] in idx]
    print(" | ".join(cols))
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0][:44]
        out = [name]
        for key, label, scale in WANT:
            if key not in idx:
                continue
            v = r[idx[key]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                out.append(v)
                continue
            u = units[idx[key]]
            if label.endswith("_MB"):
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            elif label == "dur_us":
                x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                         "ms": 1e3}[u]
            out.append(f"{x:.3g}")
        print(" | ".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
