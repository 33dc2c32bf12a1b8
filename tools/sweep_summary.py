"""Summarise tools/round_check.sh's bench sweep into a markdown table (profiles/)."""
import glob
import json
import os
import sys

d, out = sys.argv[1], sys.argv[2]
rows, brows = [], []
for f in sorted(glob.glob(os.path.join(d, "*.log"))):
    try:
        j = json.loads([x for x in open(f) if x.startswith("{")][-1])
    except Exception:
        rows.append(f"| {os.path.basename(f)[:-4]} | failed | | | | | | |")
        continue
    r, lr = j["roofline"], j["layer_roofline"]
    ph = j.get("phase_ms", {})
    top = ", ".join(f"{k} {v * 1e3:.0f}" for k, v in sorted(ph.items(), key=lambda kv: -kv[1])[:5])
    rows.append(f"| {j['config']['workload']} | {j['value'] / 1e6:.3f} M | {j['ms_per_step'] * 1e3:.0f} | "
                f"{r['bound']} {r['achieved']:.0f} {r['unit']} = {r['frac']:.2f} | {lr['frac']:.2f} | "
                f"{j['e2e']['value'] / 1e6:.2f} M | {j['clocks'].get('sm_mhz')} | {top} |")
    b = j.get("backward")
    if b:
        bp = ", ".join(f"{k} {v * 1e3:.0f}" for k, v in sorted(b["phase_ms"].items(), key=lambda kv: -kv[1])[:4])
        brows.append(f"| {j['config']['workload']} | {b['ms'] * 1e3:.0f} | {b['gemm_tflops_over_step']:.0f} | {bp} |")
hdr = ["# Bench sweep over the BASELINE configs (N = 1, EP = 1, blocking; `tools/round_check.sh`)", "",
       "value = tokens/s (device, CUDA-graph replays, L2 flushed per step); roofline = routed GEMM1 vs the "
       "measured burst bf16 peak (prefill) or HBM copy bandwidth (decode); layer = max(expert FLOPs / bf16 peak, "
       "expert weight bytes / HBM) / step time; phases in µs from instrumented replays.", "",
       "| workload | tokens/s | µs/step | GEMM1 roofline | layer roofline frac | e2e tokens/s | SM MHz | top phases (µs) |",
       "|---|---|---|---|---|---|---|---|"]
bhdr = ["", "## Backward (`fsc_moe_backward`, same layer)", "",
        "| workload | µs/step | GEMM TFLOP/s over the step | top phases (µs) |", "|---|---|---|---|"]
text = "\n".join(hdr + rows + (bhdr + brows if brows else [])) + "\n"
open(out, "w").write(text)
print(text)
