"""Summarise ncu output into profiles/ (committed evidence).

  python tools/ncu_summary.py launches gpurun_out/r01_launches.csv profiles/r01_launches.md
  python tools/ncu_summary.py full gpurun_out/r01_gemm.ncu-rep profiles/r01_ncu_gemm.md [json_out]
"""
import csv
import json
import subprocess
import sys
from collections import OrderedDict


def short(name):
    name = name.replace("void ", "")
    return name.split("(")[0]


def launches(csv_path, out_md):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    ks = [(int(r[ii]), short(r[ki]), float(r[vi]) / 1e3) for r in rows[hi + 1:] if len(r) == len(h)]
    # one step = from one router launch (its first kernel: the W' quantisation of the
    # tensor-core router, or the SIMT router's prescale) to the next
    starts = [i for i, (_, n, _) in enumerate(ks) if "router_tc_quant_w" in n or "router_prescale" in n]
    step = ks[starts[-2]:starts[-1]] if len(starts) >= 2 else ks
    tot = sum(t for _, _, t in step)
    lines = [f"# Launch list of one bench step (ncu gpu__time_duration.sum, --clock-control none)",
             "", f"source: `{csv_path}` (serialised, cold-cache per launch; compare shares, not absolutes)", "",
             "| # | kernel | us | share |", "|---|---|---|---|"]
    for i, (_, n, t) in enumerate(step):
        lines.append(f"| {i} | `{n}` | {t:.1f} | {100 * t / tot:.1f}% |")
    lines.append(f"| | **total** | **{tot:.1f}** | 100% |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_active_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("lts__t_sectors_op_read.sum", "l2_read_sectors"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster_x"),
    ("sm__cycles_active.avg", "sm_cycles_active"),
])


def full(rep, out_md, json_out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m, key in METRICS.items():
            if m in h:
                i = h.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[i]
                if isinstance(v, float) and u in ("Mbyte", "Gbyte", "Kbyte", "byte"):
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                    u = "byte"
                if isinstance(v, float) and u in ("usecond", "msecond", "nsecond"):
                    v = v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}[u]
                    u = "us"
                d[key] = v
        out.append(d)
    lines = [f"# ncu --set full summary: `{rep}`", "", "| kernel | us | DRAM read MB | DRAM write MB | tensor pipe % "
             "| SM thr % | DRAM thr % | regs | grid | cluster |", "|---|---|---|---|---|---|---|---|---|---|"]
    for d in out:
        lines.append(f"| `{d['kernel']}` | {d.get('duration', 0):.1f} | {d.get('dram_read', 0) / 1e6:.1f} | "
                     f"{d.get('dram_write', 0) / 1e6:.1f} | {d.get('tensor_pipe_active_pct', 0):.1f} | "
                     f"{d.get('sm_throughput_pct', 0):.1f} | {d.get('dram_throughput_pct', 0):.1f} | "
                     f"{d.get('registers', '')} | {d.get('grid', '')} | {d.get('cluster_x', '')} |")
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if json_out:
        json.dump(out, open(json_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
