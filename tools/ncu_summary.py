"""Summarise the ncu captures of tools/ncu_profile.sh into profiles/ (JSON + markdown).

usage: python tools/ncu_summary.py gpurun_out/TAG profiles/ncu_summary.json profiles/ncu_summary_r01.md
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

src, out_json, out_md = Path(sys.argv[1]), Path(sys.argv[2]), Path(sys.argv[3])
WANT = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "l2_sectors": ("lts__t_sectors.sum", 1.0),
    "l2_to_sm_bytes": ("l1tex__m_xbar2l1tex_read_bytes.sum", 1.0),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_pct_peak": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l1tex_pct_peak": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    "sm_pct_peak": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TUNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


res = {}
for rep in sorted(src.glob("*.ncu-rep")):
    h, u, v = raw(rep)
    d = {"kernel": v[h.index("Kernel Name")][:80] if "Kernel Name" in h else ""}
    for key, (metric, scale) in WANT.items():
        name = metric if metric in h else next((n for n in h if n.endswith("." + metric)), None)
        if name is None:
            continue
        i = h.index(name)
        try:
            x = float(v[i].replace(",", ""))
        except ValueError:
            continue
        unit = u[i]
        if key == "duration_us":
            x = x * TUNIT.get(unit, 1.0)
        elif unit in UNIT and key.endswith("bytes"):
            x = x * UNIT[unit]
        d[key] = round(x, 3)
    if "l2_sectors" in d:
        d["l2_bytes"] = d["l2_sectors"] * 32
    if "dram_read_bytes" in d and "dram_write_bytes" in d:
        d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
    res[rep.stem] = d
summary = {"source": str(src), "note": "ncu --set full --clock-control none --cache-control all (L2 flushed before "
           "every replay pass: cold-cache DRAM bytes, as in the flushed bench step), one launch of the bench step "
           "(tools/ncu_profile.sh); bytes are per launch",
           "kernels": res,
           "dram_bytes_per_launch": {k: v.get("dram_bytes") for k, v in res.items()}}
out_json.write_text(json.dumps(summary, indent=1))
lines = ["| capture | kernel | us | DRAM MB | L2 MB | L2->SM MB | L2->SM TB/s | DRAM %pk | L2 %pk | L1 %pk | tensor % | "
         "warps % | regs |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for k, d in res.items():
    lines.append(f"| {k} | `{d.get('kernel', '')[:40]}` | {d.get('duration_us', 0):.1f} | "
                 f"{d.get('dram_bytes', 0) / 1e6:.1f} | {d.get('l2_bytes', 0) / 1e6:.1f} | "
                 f"{d.get('l2_to_sm_bytes', 0) / 1e6:.1f} | "
                 f"{d.get('l2_to_sm_bytes', 0) / max(d.get('duration_us', 1), 1e-9) / 1e6:.2f} | {d.get('dram_pct_peak', 0):.1f} | "
                 f"{d.get('l2_pct_peak', 0):.1f} | {d.get('l1tex_pct_peak', 0):.1f} | {d.get('tensor_pipe_pct', 0):.1f} | "
                 f"{d.get('warps_active_pct', 0):.1f} | {d.get('registers', 0):.0f} |")
out_md.write_text("\n".join(lines) + "\n")
print("\n".join(lines))
