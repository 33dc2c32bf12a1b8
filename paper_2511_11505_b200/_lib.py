"""ctypes binding of libfsc (include/fsc.h) — argument marshalling only.

Every step of the MoE forward runs inside libfsc's CUDA kernels; this module
only converts torch tensors to device pointers and status codes to
exceptions. There is no fallback: if libfsc.so is missing or a call fails,
an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSC_LIB", os.path.join(HERE, "libfsc.so"))

FSC_OK, FSC_ERR_CONFIG, FSC_ERR_SHAPE, FSC_ERR_CUDA, FSC_ERR_COMM, FSC_ERR_NONFINITE, FSC_ERR_STATE = 0, -1, -2, -3, -4, -5, -6
FSC_REGULAR, FSC_HYBRID = 0, 1
FSC_BLOCKING, FSC_OVERLAPPED = 0, 1
FSC_EP_ALLTOALL, FSC_EP_ALLREDUCE = 0, 1
FSC_COMBINE_STREAM, FSC_COMBINE_FUSED = 0, 1
FSC_BLOCKING_REGULAR_PLUS, FSC_BLOCKING_SERIAL = 0, 1
SPIN_PHASES = ("gate", "dispatch", "qkv", "core", "routed", "combine", "shared")   # FSC_SPIN_* order
EPI_BF16, EPI_SWIGLU, EPI_RESID_F32 = 0, 1, 2

_STATUS = {FSC_ERR_CONFIG: "CONFIG", FSC_ERR_SHAPE: "SHAPE", FSC_ERR_CUDA: "CUDA", FSC_ERR_COMM: "COMM",
           FSC_ERR_NONFINITE: "NONFINITE", FSC_ERR_STATE: "STATE"}


class FscError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fsc error {code} ({_STATUS.get(code, '?')}): {msg}")
        self.code = code


class MoeConfig(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("n_experts", ctypes.c_int), ("top_k", ctypes.c_int), ("ffn", ctypes.c_int),
                ("shared_ffn", ctypes.c_int), ("max_tokens", ctypes.c_int), ("rms_eps", ctypes.c_float)]


class MoeWeightsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("gamma", "w_router", "w1", "w2", "w3", "ws1", "ws2", "ws3")]


class MoeDebugC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("topk_idx", "topk_w", "counts", "pos", "logits", "shared_out",
                                               "routed_out", "n_refined", "ep_counts", "recv_counts", "recv_src")]


class MoeGradsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("dx", "dgamma", "dw_router", "dw1", "dw2", "dw3", "dws1", "dws2",
                                               "dws3")]


class AttnWeightsC(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_void_p), ("w_qkv", ctypes.c_void_p), ("w_o", ctypes.c_void_p),
                ("n_heads", ctypes.c_int), ("n_kv_heads", ctypes.c_int), ("head_dim", ctypes.c_int),
                ("rope_theta", ctypes.c_float)]


class ActCacheC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("attn_in", "mlp_in", "attn_out", "shared_out", "routed_out", "o")]


OVERLAP_CB = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_long
_SIGS = {
    "fsc_bootstrap_size": (ctypes.c_size_t, []),
    "fsc_init": (_I, [ctypes.POINTER(_P), _I, _I, _I, ctypes.POINTER(MoeConfig)]),
    "fsc_bootstrap_export": (_I, [_P, _P]),
    "fsc_bootstrap_import": (_I, [_P, _P]),
    "fsc_finalize": (_I, [_P]),
    "fsc_last_error": (ctypes.c_char_p, [_P]),
    "fsc_set_gemm_ctas": (_I, [_P, _I]),
    "fsc_set_gemm_cta_group": (_I, [_P, _I]),
    "fsc_set_gemm_gather": (_I, [_P, _I]),
    "fsc_set_fused_unpermute": (_I, [_P, _I]),
    "fsc_set_router_int8": (_I, [_P, _I]),
    "fsc_set_router_f64": (_I, [_P, _I]),
    "fsc_set_gemm_dynamic": (_I, [_P, _I]),
    "fsc_set_ep_mode": (_I, [_P, _I]),
    "fsc_set_dispatch_fp8": (_I, [_P, _I]),
    "fsc_set_debug_checks": (_I, [_P, _I]),
    "fsc_set_combine_mode": (_I, [_P, _I]),
    "fsc_set_blocking_mode": (_I, [_P, _I]),
    "fsc_set_comm_ctas": (_I, [_P, _I]),
    "fsc_set_a2a_zero_bytes": (_I, [_P, _I]),
    "fsc_set_spin_schedule": (_I, [_P, _P]),
    "fsc_set_delay_fuzz": (_I, [_P, ctypes.c_uint, ctypes.c_longlong]),
    "fsc_timeline": (_I, [_P, _P, _P, _P, _P, _I]),
    "fsc_set_timing": (_I, [_P, _I]),
    "fsc_set_timing_mask": (_I, [_P, ctypes.c_uint]),
    "fsc_get_timings": (_I, [_P, ctypes.POINTER(ctypes.c_float), _I]),
    "fsc_launch_count": (ctypes.c_long, []),
    "fsc_timing_log": (_I, [_P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_float), _I]),
    "fsc_moe_forward_blocking": (_I, [_P, ctypes.POINTER(MoeWeightsC), _I, _P, _P, ctypes.POINTER(MoeDebugC), _P]),
    "fsc_moe_forward_blocking_host": (_I, [_P, ctypes.POINTER(MoeWeightsC), _I, _P, _P, _P]),
    "fsc_moe_forward_host_async": (_I, [_P, ctypes.POINTER(MoeWeightsC), _I, _P, _P, _P]),
    "fsc_host_flush": (_I, [_P]),
    "fsc_moe_forward_farskip": (_I, [_P, ctypes.POINTER(MoeWeightsC), _I, _P, _P, OVERLAP_CB, _P,
                                     ctypes.POINTER(_P), ctypes.POINTER(MoeDebugC), _P]),
    "fsc_moe_wait": (_I, [_P, _P, _P, _P, _P]),
    "fsc_layer_stack_forward": (_I, [_P, ctypes.POINTER(AttnWeightsC), ctypes.POINTER(MoeWeightsC), _I, _I, _I,
                                     ctypes.POINTER(_I), _I, _P, _P, ctypes.POINTER(ActCacheC), _P]),
    "fsc_op_router": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "fsc_op_perm_maps": (_I, [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "fsc_op_permute": (_I, [_P, _P, _P, _P, _I, _I, _P]),
    "fsc_op_grouped_gemm": (_I, [_P, _I, _P, _L, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P]),
    "fsc_op_grouped_gemm_gather": (_I, [_P, _I, _P, _L, _P, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P]),
    "fsc_op_unpermute": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P]),
    "fsc_op_attention": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P]),
    "fsc_moe_backward": (_I, [_P, ctypes.POINTER(MoeWeightsC), _I, _P, _P, ctypes.POINTER(MoeGradsC), _P]),
    "fsc_op_gemm_dgrad": (_I, [_P, _I, _P, _L, _P, _P, _L, _I, _P, _I, _I, _I, _I, _P, _P, _P]),
    "fsc_op_gemm_swiglu_bwd": (_I, [_P, _P, _L, _P, _P, _I, _P, _I, _I, _I, _P, _P, _P, _P, _P, _I, _P]),
    "fsc_op_gemm_wgrad": (_I, [_P, _P, _I, _I, _I, _I, _P, _L, _L, _I, _P, _L, _I, _P, _I, _P]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfsc.so (built by paper_2511_11505_b200.build); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libfsc.so not found at {path}: run `python -m paper_2511_11505_b200.build` "
                          "(there is no fallback path)")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def ptr(t) -> Optional[int]:
    """Device pointer of a tensor (or an int / None passthrough)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def cur_stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


class MoeWeights:
    """Keeps the tensors alive and exposes the C struct."""

    def __init__(self, gamma, w_router, w1, w2, w3, ws1=None, ws2=None, ws3=None):
        self.tensors = (gamma, w_router, w1, w2, w3, ws1, ws2, ws3)
        self.c = MoeWeightsC(*[ptr(t) for t in self.tensors])


class MoeDebug:
    def __init__(self, **kw):
        self.tensors = kw
        self.c = MoeDebugC(**{k: ptr(v) for k, v in kw.items()})


class AttnWeights:
    def __init__(self, gamma, w_qkv, w_o, n_heads, n_kv_heads, head_dim, rope_theta=10000.0):
        self.tensors = (gamma, w_qkv, w_o)
        self.c = AttnWeightsC(ptr(gamma), ptr(w_qkv), ptr(w_o), n_heads, n_kv_heads, head_dim, rope_theta)


def exchange_blobs(blob: bytes, group=None):
    """All-gather one bytes blob per rank, returned in rank order (torch.distributed)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


class Context:
    """One EP rank's libfsc context."""

    def __init__(self, d, n_experts, top_k, ffn, shared_ffn, max_tokens, rank=0, ep_size=1, device=0,
                 rms_eps=1e-6):
        self.lib = load()
        self.cfg = MoeConfig(d, n_experts, top_k, ffn, shared_ffn, max_tokens, rms_eps)
        h = _P()
        rc = self.lib.fsc_init(ctypes.byref(h), rank, ep_size, device, ctypes.byref(self.cfg))
        self.h = h
        if rc:
            msg = self.lib.fsc_last_error(h).decode() if h.value else "fsc_init failed"
            if h.value:
                self.lib.fsc_finalize(h)
                self.h = _P()
            raise FscError(rc, msg)
        self._pending_cb = None

    # -- lifecycle
    def close(self):
        if self.h and self.h.value:
            self.lib.fsc_finalize(self.h)
            self.h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc):
        if rc:
            raise FscError(rc, self.lib.fsc_last_error(self.h).decode())

    def bootstrap_export(self) -> bytes:
        n = self.lib.fsc_bootstrap_size()
        buf = ctypes.create_string_buffer(max(n, 1))
        self._ck(self.lib.fsc_bootstrap_export(self.h, buf))
        return buf.raw[:n]

    def connect(self, group=None):
        """Bootstrap the EP transport: every rank exports its peer-region handle,
        the handles are all-gathered in rank order over torch.distributed (host
        plumbing only), and every rank maps its peers'."""
        blob = self.bootstrap_export()
        self.bootstrap_import(exchange_blobs(blob, group))

    def bootstrap_import(self, blobs: Sequence[bytes]):
        data = b"".join(blobs)
        buf = ctypes.create_string_buffer(data, max(len(data), 1))
        self._ck(self.lib.fsc_bootstrap_import(self.h, buf))

    PHASES = ("router", "perm_maps", "dispatch", "gemm1", "gemm2", "combine", "shared1", "shared2", "unpermute",
              "dispatch_stall", "combine_wait", "attn_a", "attn_b")
    STREAMS = ("compute", "comm", "aux")

    def set_timing(self, enable: bool):
        self._ck(self.lib.fsc_set_timing(self.h, int(enable)))

    def set_timing_mask(self, phases):
        """Time only the named phases (see PHASES); [] disables timing."""
        mask = 0
        for n in phases:
            mask |= 1 << self.PHASES.index(n)
        self._ck(self.lib.fsc_set_timing_mask(self.h, mask))

    def timings(self) -> dict:
        """Per-phase ms of the last MoE call (phases not run are omitted)."""
        buf = (ctypes.c_float * len(self.PHASES))()
        rc = self.lib.fsc_get_timings(self.h, buf, len(self.PHASES))
        if rc < 0:
            self._ck(rc)
        return {n: buf[i] for i, n in enumerate(self.PHASES) if buf[i] >= 0}

    def timing_log(self, cap: int = 1024):
        """[(phase_name, ms)] for every timed phase instance since set_timing(True)."""
        ph = (ctypes.c_int * cap)()
        ms = (ctypes.c_float * cap)()
        n = self.lib.fsc_timing_log(self.h, ph, ms, cap)
        if n < 0:
            self._ck(n)
        return [(self.PHASES[ph[i]], ms[i]) for i in range(n)]

    def timeline(self, cap: int = 4096):
        """[(phase, stream, t0_ms, dur_ms)] of every logged phase instance (fsc_timeline)."""
        ph = (ctypes.c_int * cap)()
        st = (ctypes.c_int * cap)()
        t0 = (ctypes.c_float * cap)()
        du = (ctypes.c_float * cap)()
        n = self.lib.fsc_timeline(self.h, ph, st, t0, du, cap)
        if n < 0:
            self._ck(n)
        return [(self.PHASES[ph[i]], self.STREAMS[st[i]], t0[i], du[i]) for i in range(n)]

    def set_combine_mode(self, mode: int):
        """FSC_COMBINE_STREAM (comm-stream push after the down GEMM) or FSC_COMBINE_FUSED."""
        self._ck(self.lib.fsc_set_combine_mode(self.h, mode))

    def set_blocking_mode(self, mode: int):
        """FSC_BLOCKING_REGULAR_PLUS or FSC_BLOCKING_SERIAL (fsc_moe_forward_blocking at EP > 1)."""
        self._ck(self.lib.fsc_set_blocking_mode(self.h, mode))

    def set_comm_ctas(self, n: int):
        self._ck(self.lib.fsc_set_comm_ctas(self.h, n))

    def set_a2a_zero_bytes(self, on: bool):
        """Measurement instrument: all-to-all without payload rows (flags and counts only)."""
        self._ck(self.lib.fsc_set_a2a_zero_bytes(self.h, int(on)))

    def set_spin_schedule(self, unit_ns):
        """{phase: ns} over SPIN_PHASES (spin kernels instead of the real work), or None."""
        if unit_ns is None:
            self._ck(self.lib.fsc_set_spin_schedule(self.h, None))
            return
        arr = (ctypes.c_longlong * len(SPIN_PHASES))(*[int(unit_ns[p]) for p in SPIN_PHASES])
        self._ck(self.lib.fsc_set_spin_schedule(self.h, arr))

    def set_delay_fuzz(self, seed: int, max_ns: int):
        self._ck(self.lib.fsc_set_delay_fuzz(self.h, seed, max_ns))

    def launch_count(self) -> int:
        return int(self.lib.fsc_launch_count())

    def set_gemm_cta_group(self, cg: int):
        self._ck(self.lib.fsc_set_gemm_cta_group(self.h, cg))

    def set_gemm_gather(self, on: bool):
        """EP = 1: fuse the permute into GEMM1 (TMA gather4 of the xn rows)."""
        self._ck(self.lib.fsc_set_gemm_gather(self.h, int(on)))

    def set_dispatch_fp8(self, on: bool):
        """EP > 1 all-to-all: FP8 e4m3 dispatch payload with per-128-column scales. Call before connect()."""
        self._ck(self.lib.fsc_set_dispatch_fp8(self.h, int(on)))

    def set_ep_mode(self, mode: int):
        """FSC_EP_ALLTOALL (Dispatch / Combine) or FSC_EP_ALLREDUCE (replicated tokens,
        P:215-217). Call before connect()."""
        self._ck(self.lib.fsc_set_ep_mode(self.h, mode))

    def set_gemm_dynamic(self, on):
        """Grouped-GEMM tile schedule: True (dynamic), False (static stride) or None (auto:
        dynamic at EP > 1)."""
        self._ck(self.lib.fsc_set_gemm_dynamic(self.h, -1 if on is None else int(on)))

    def set_router_int8(self, on):
        """Router on the tensor cores (the fused exact int8-digit kernel; E <= 128, d % 128 == 0,
        k <= 8): True / None (auto, the default: wherever the shape allows) or False (the fp32
        SIMT router)."""
        self._ck(self.lib.fsc_set_router_int8(self.h, -1 if on is None else int(on)))

    def set_router_f64(self, on):
        """fp64 small-batch router (router_f64_kernel): True (every call), False (never) or
        None (auto, the default: T x EP x d <= 2.7e8 unless the fp32 SIMT router was selected)."""
        self._ck(self.lib.fsc_set_router_f64(self.h, -1 if on is None else int(on)))

    def set_fused_unpermute(self, on):
        """Blocking EP = 1: gate-weighted unpermute fused into the down GEMM epilogue
        (True / False; None = auto: top-1 routing only)."""
        self._ck(self.lib.fsc_set_fused_unpermute(self.h, -1 if on is None else int(on)))

    def set_debug_checks(self, on: bool):
        """Finiteness check of every output (synchronises; FSC_ERR_NONFINITE on failure)."""
        self._ck(self.lib.fsc_set_debug_checks(self.h, int(on)))

    def set_gemm_ctas(self, n: int):
        self._ck(self.lib.fsc_set_gemm_ctas(self.h, n))

    # -- MoE
    def moe_forward_blocking(self, w: MoeWeights, x_in, out, dbg: Optional[MoeDebug] = None, stream=None):
        T = x_in.shape[0]
        self._ck(self.lib.fsc_moe_forward_blocking(self.h, ctypes.byref(w.c), T, ptr(x_in), ptr(out),
                                                   ctypes.byref(dbg.c) if dbg else None,
                                                   stream if stream is not None else cur_stream()))

    def moe_forward_blocking_host(self, w: MoeWeights, x_host, out_host, stream=None):
        T = x_host.shape[0]
        self._ck(self.lib.fsc_moe_forward_blocking_host(self.h, ctypes.byref(w.c), T, ptr(x_host), ptr(out_host),
                                                        stream if stream is not None else cur_stream()))

    def moe_forward_host_async(self, w: MoeWeights, x_host, out_host, stream=None):
        T = x_host.shape[0]
        self._ck(self.lib.fsc_moe_forward_host_async(self.h, ctypes.byref(w.c), T, ptr(x_host), ptr(out_host),
                                                     stream if stream is not None else cur_stream()))

    def host_flush(self):
        self._ck(self.lib.fsc_host_flush(self.h))

    def moe_forward_farskip(self, w: MoeWeights, x_in, partial_inout, callback=None,
                            dbg: Optional[MoeDebug] = None, stream=None):
        T = x_in.shape[0]
        if callback is not None:
            cb = OVERLAP_CB(lambda user, phase, s: callback(phase, s))
        else:
            cb = OVERLAP_CB()
        self._pending_cb = cb
        h = _P()
        self._ck(self.lib.fsc_moe_forward_farskip(self.h, ctypes.byref(w.c), T, ptr(x_in), ptr(partial_inout), cb,
                                                  None, ctypes.byref(h), ctypes.byref(dbg.c) if dbg else None,
                                                  stream if stream is not None else cur_stream()))
        return h

    def moe_wait(self, handle, partial_in, full_out, stream=None):
        self._ck(self.lib.fsc_moe_wait(self.h, handle, ptr(partial_in), ptr(full_out),
                                       stream if stream is not None else cur_stream()))

    def layer_stack_forward(self, attn: Sequence[AttnWeights], moe: Sequence[MoeWeights], T: int, seq_len: int,
                            modes: Sequence[int], schedule: int, o0, oL, cache=None, stream=None):
        L = len(moe)
        aw = (AttnWeightsC * L)(*[a.c for a in attn])
        mw = (MoeWeightsC * L)(*[m.c for m in moe])
        md = (ctypes.c_int * L)(*modes)
        cc = None
        if cache is not None:
            cc = (ActCacheC * L)(*[ActCacheC(**{k: ptr(v) for k, v in c.items()}) for c in cache])
        self._ck(self.lib.fsc_layer_stack_forward(self.h, aw, mw, L, T, seq_len, md, schedule, ptr(o0), ptr(oL), cc,
                                                  stream if stream is not None else cur_stream()))

    # -- backward
    def moe_backward(self, w: MoeWeights, x_in, grad_out, grads: dict, stream=None):
        """grads: {"dx": ..., optional "dgamma", "dw_router", "dw1", "dw2", "dw3", "dws1", "dws2", "dws3"}
        (fp32 device tensors, written)."""
        T = x_in.shape[0]
        g = MoeGradsC(**{k: ptr(v) for k, v in grads.items()})
        self._ck(self.lib.fsc_moe_backward(self.h, ctypes.byref(w.c), T, ptr(x_in), ptr(grad_out), ctypes.byref(g),
                                           stream if stream is not None else cur_stream()))

    def op_gemm_dgrad(self, epi, A, B0, B1, b_group_rows, G, counts, m_total, N, K, kb_split, out, resid=None,
                      stream=None):
        self._ck(self.lib.fsc_op_gemm_dgrad(self.h, epi, ptr(A), A.shape[0], ptr(B0), ptr(B1), b_group_rows, G,
                                            ptr(counts), m_total, N, K, kb_split, ptr(out), ptr(resid),
                                            stream if stream is not None else cur_stream()))

    def op_gemm_swiglu_bwd(self, A, B0, B1, G, counts, m_total, N, K, dh, row_gate, duv, hg, dg_part=None,
                           dg_ld=0, stream=None):
        self._ck(self.lib.fsc_op_gemm_swiglu_bwd(self.h, ptr(A), A.shape[0], ptr(B0), ptr(B1), G, ptr(counts),
                                                 m_total, N, K, ptr(dh), ptr(row_gate), ptr(duv), ptr(hg),
                                                 ptr(dg_part), dg_ld, stream if stream is not None else cur_stream()))

    def op_gemm_wgrad(self, counts, G, m_total, N1, N2, A, lda, a_col0, B, ldb, b_col0, out, accumulate=False,
                      stream=None):
        self._ck(self.lib.fsc_op_gemm_wgrad(self.h, ptr(counts), G, m_total, N1, N2, ptr(A), A.shape[0], lda, a_col0,
                                            ptr(B), ldb, b_col0, ptr(out), int(accumulate),
                                            stream if stream is not None else cur_stream()))

    # -- op level
    def op_router(self, x, gamma, w_router, k, xn, topk_idx, topk_w, logits=None, n_refined=None, stream=None):
        T, d = x.shape
        E = w_router.shape[0]
        self._ck(self.lib.fsc_op_router(self.h, ptr(x), ptr(gamma), ptr(w_router), T, d, E, k, ptr(xn), ptr(topk_idx),
                                        ptr(topk_w), ptr(logits), ptr(n_refined),
                                        stream if stream is not None else cur_stream()))

    def op_perm_maps(self, topk_idx, E, counts, offsets, pos, src_row, stream=None):
        T, k = topk_idx.shape
        self._ck(self.lib.fsc_op_perm_maps(self.h, ptr(topk_idx), T, k, E, ptr(counts), ptr(offsets), ptr(pos),
                                           ptr(src_row), stream if stream is not None else cur_stream()))

    def op_permute(self, xn, src_row, xs, stream=None):
        R, d = xs.shape
        self._ck(self.lib.fsc_op_permute(self.h, ptr(xn), ptr(src_row), ptr(xs), R, d,
                                         stream if stream is not None else cur_stream()))

    def op_grouped_gemm(self, epi, A, B0, B1, G, counts, m_total, N, K, out, resid=None, stream=None):
        self._ck(self.lib.fsc_op_grouped_gemm(self.h, epi, ptr(A), A.shape[0], ptr(B0), ptr(B1), G, ptr(counts),
                                              m_total, N, K, ptr(out), ptr(resid),
                                              stream if stream is not None else cur_stream()))

    def op_grouped_gemm_gather(self, epi, A, a_idx, B0, B1, G, counts, m_total, N, K, out, resid=None, stream=None):
        """Row r of the grouped problem reads A[a_idx[r]] (TMA gather4 in the GEMM producer)."""
        self._ck(self.lib.fsc_op_grouped_gemm_gather(self.h, epi, ptr(A), A.shape[0], ptr(a_idx), ptr(B0), ptr(B1), G,
                                                     ptr(counts), m_total, N, K, ptr(out), ptr(resid),
                                                     stream if stream is not None else cur_stream()))

    def op_attention(self, qkv, out, Hq, Hkv, hd, seq_len, stream=None):
        self._ck(self.lib.fsc_op_attention(self.h, ptr(qkv), ptr(out), qkv.shape[0], Hq, Hkv, hd, seq_len,
                                           stream if stream is not None else cur_stream()))

    def op_unpermute(self, y, pos, w, resid, out, stream=None):
        T, k = pos.shape
        d = out.shape[1]
        self._ck(self.lib.fsc_op_unpermute(self.h, ptr(y), ptr(pos), ptr(w), ptr(resid), ptr(out), T, k, d,
                                           stream if stream is not None else cur_stream()))
