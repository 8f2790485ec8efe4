"""Key metrics of ncu --set full captures as a markdown table.

    python tools/ncu_summary.py gpurun_out/prof/*.ncu-rep
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time (us)", 1e-3),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1e-6),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak", 1),
    ("sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
     "int8 tensor % peak", 1),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy (IMAD) pipe %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__registers_per_thread", "regs", 1),
]


def metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None, {}
    h, units, vals = rows[0], rows[1], rows[2]
    name = vals[h.index("Kernel Name")] if "Kernel Name" in h else path
    d = {}
    for key, _, _ in WANT:
        if key in h:
            v = vals[h.index(key)].replace(",", "")
            u = units[h.index(key)]
            try:
                x = float(v)
            except ValueError:
                continue
            # normalise units reported by ncu
            if key == "gpu__time_duration.sum":
                x = x * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
                         "s": 1e9, "second": 1e9}.get(u, 1)
            elif key.startswith("dram__bytes"):
                x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            d[key] = x
    return name, d


print("| kernel | " + " | ".join(lbl for _, lbl, _ in WANT) + " |")
print("|---|" + "---|" * len(WANT))
for p in sys.argv[1:]:
    name, d = metrics(p)
    cells = []
    for key, _, scale in WANT:
        v = d.get(key)
        cells.append("" if v is None else (f"{v * scale:.3g}" if scale != 1 else f"{v:.4g}"))
    print(f"| `{(name or p)[:60]}` | " + " | ".join(cells) + " |")
