"""A/B of the GEMM epilogue store mode (FSC_GEMM_STAGE_ROWS=0/1) in one GPU session."""
import os
import subprocess
import sys

for rep in range(2):
    for v in ("0", "1"):
        env = dict(os.environ, FSC_GEMM_STAGE_ROWS=v)
        out = subprocess.run([sys.executable, "tools/gemm_bench.py"], env=env, capture_output=True, text=True).stdout
        rows = [l for l in out.splitlines() if l.startswith(("DS gemm1", "DS gemm2", "DS shared1", "qwen3 gemm1", "qwen3 gemm2",
                                                              "scout gemm1"))]
        print(f"stage={v}", " | ".join(f"{l.split()[0]} {l.split()[1]} {l.split(':')[-1].split('us')[0].strip()}"
                                       for l in rows if "cg=2" in l), flush=True)
