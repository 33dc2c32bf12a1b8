"""CPU checks of the C-ABI boundary: libfsc.so builds for sm_100a, exports
every symbol include/fsc.h declares, rejects bad configs before touching the
GPU, and carries the tcgen05 / TMA instructions in its SASS."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsc.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2511_11505_b200 import build as b
    b.build()
    from paper_2511_11505_b200 import _lib
    return _lib.load()


def declared():
    src = open(HEADER).read()
    return re.findall(r"^FSC_API [^(]*?\b(fsc_\w+)\(", src, flags=re.M)


def test_header_declares_the_survey_entry_points():
    names = set(declared())
    for n in ["fsc_init", "fsc_finalize", "fsc_last_error", "fsc_moe_forward_blocking", "fsc_moe_forward_farskip",
              "fsc_moe_wait", "fsc_layer_stack_forward"]:
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2511_11505_b200", "libfsc.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (\w+)", out))
    assert set(declared()) <= exported
    # nothing but the C ABI is exported (C++ internals stay hidden)
    assert all(n.startswith("fsc_") for n in exported), sorted(n for n in exported if not n.startswith("fsc_"))


@pytest.mark.parametrize("bad", [
    dict(d=100), dict(n_experts=0), dict(n_experts=129), dict(top_k=0), dict(top_k=5), dict(ffn=100),
    dict(shared_ffn=10), dict(ep=3), dict(rank=2, ep=2), dict(max_tokens=-1)])
def test_init_rejects_bad_config_without_gpu(lib, bad):
    from paper_2511_11505_b200._lib import FSC_ERR_CONFIG, MoeConfig
    c = dict(d=64, n_experts=4, top_k=2, ffn=128, shared_ffn=0, max_tokens=32, rank=0, ep=1)
    c.update(bad)
    cfg = MoeConfig(c["d"], c["n_experts"], c["top_k"], c["ffn"], c["shared_ffn"], c["max_tokens"], 1e-6)
    h = ctypes.c_void_p()
    assert lib.fsc_init(ctypes.byref(h), c["rank"], c["ep"], 0, ctypes.byref(cfg)) == FSC_ERR_CONFIG
    assert not h.value


def test_null_context_is_an_error_not_a_crash(lib):
    assert lib.fsc_finalize(None) == 0
    assert lib.fsc_moe_forward_blocking(None, None, 0, None, None, None, None) < 0
    assert lib.fsc_last_error(None) == b"null context"


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="no cuobjdump")
def test_sass_is_blackwell_native(lib):
    so = os.path.join(ROOT, "paper_2511_11505_b200", "libfsc.so")
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    elf = subprocess.run([cuobjdump, "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in elf
    sass = subprocess.run([cuobjdump, "-sass", so], capture_output=True, text=True).stdout
    # split per function; the grouped GEMM (every expert / shared / projection GEMM)
    # must be tcgen05 + TMA, with no legacy mma.sync
    funcs = re.split(r"\n\s*Function : ", sass)
    gemm = [f for f in funcs if f.startswith("_ZN3fsc19grouped_gemm_kernel")]
    assert len(gemm) >= 16, len(gemm)
    for f in gemm:
        name = f.split()[0]
        assert "UTCHMMA" in f or "UTCMMA" in f, f"tcgen05.mma missing in {name}"
        assert "UTMALDG" in f, f"TMA load missing in {name}"
        assert "LDTM" in f, f"tcgen05.ld missing in {name}"
        assert not re.search(r"\bHMMA\b", f), f"legacy mma.sync in {name}"
