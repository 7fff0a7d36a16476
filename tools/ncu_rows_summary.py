"""Table of the key ncu counters per row kernel (tools/ncu_rows.sh output)."""
import csv
import io
import sys
from pathlib import Path

tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
cols = [("gpu__time_duration.sum", "ms", 1e-6), ("smsp__inst_executed.sum", "Ginst", 1e-9),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes/32", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%", 1),
        ("dram__bytes_read.sum", "DRAMrd GB", 1e-9), ("dram__bytes_write.sum", "DRAMwr GB", 1e-9),
        ("launch__registers_per_thread", "regs", 1), ("launch__shared_mem_per_block_dynamic", "smem KB", 1)]
print(f"{'config':14s} {'kernel':16s} " + " ".join(f"{c[1]:>10s}" for c in cols))
for f in sorted(Path("gpurun_out").glob(f"{tag}_ncu_*.csv")):
    text = f.read_text()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    if not lines:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr = rows[0]
    vals = {}
    kname = "?"
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", kname).split("<")[0].split("(")[0].split("::")[-1]
        name, unit, v = d.get("Metric Name"), d.get("Metric Unit"), d.get("Metric Value", "").replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        scale = {"msecond": 1e6, "usecond": 1e3, "second": 1e9, "nsecond": 1, "Gbyte": 1e9, "Mbyte": 1e6,
                 "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(unit, 1)
        vals[name] = v * scale
    cfg = f.stem[len(tag) + 5:]
    out = []
    for name, _, sc in cols:
        v = vals.get(name)
        if name == "launch__shared_mem_per_block_dynamic" and v is not None:
            v = v / 1e3
            sc = 1
        out.append(f"{v * sc:10.3f}" if v is not None else f"{'-':>10s}")
    print(f"{cfg:14s} {kname[:16]:16s} " + " ".join(out))
