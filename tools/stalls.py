"""Top SASS lines by warp-stall samples from an ncu report (source page).
usage: python tools_stalls.py REPORT KERNEL_REGEX [N] [--mangled]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
if kern.startswith("#"):                     # '#3' = the 4th profiled launch
    cmd += ["--launch-skip", kern[1:], "--launch-count", "1"]
else:
    cmd += ["--kernel-name", f"regex:{kern}"]
if "--mangled" in sys.argv:
    cmd[5:5] = ["--print-kernel-base", "mangled"]
lines = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(lines))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] not in ("Address", "Kernel Name")]
si, ci, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
seen = {}
for r in data:                                    # one entry per address (multiple launches repeat)
    a = r[0]
    v = float(r[ci] or 0)
    if a in seen:
        seen[a][0] += v
    else:
        seen[a] = [v, r[si].strip()[:90], r[ei]]
tot = sum(v[0] for v in seen.values())
print(f"total samples {tot:.0f}")
for a, (v, s, e) in sorted(seen.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * v / max(tot, 1):5.1f}% {a[-5:]} {s:90s} exec={e}")
