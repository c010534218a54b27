"""Thin ctypes binding of libbaatt.so (include/ba_attn.h) for torch tensors.

Argument marshalling only: torch supplies device memory and the current CUDA
stream; every step of the path runs in the library's kernels.  There is no
CPU or library fallback — if the extension is missing or a call fails, this
module raises.

Names follow the C ABI: ba_select, ba_sparse_attn, ba_attention,
ba_dense_attn, ba_attention_host.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BA_LIB_PATH") or os.path.join(HERE, "libbaatt.so")  # override: A/B builds only

BA_DTYPE_BF16, BA_DTYPE_FP32 = 0, 1
SORT = {"none": 0, "q": 1, "k": 2, "qk": 3}
COMP = {"none": 0, "diag": 1, "exact": 2}
SELECT_TOPK, SELECT_TOPP = 0, 1


class BaError(RuntimeError):
    pass


class Problem(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("heads_q", ctypes.c_int32), ("heads_kv", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("len_q", ctypes.c_int64), ("len_k", ctypes.c_int64),
                ("block_size", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("q_stride", ctypes.c_int64 * 3), ("k_stride", ctypes.c_int64 * 3),
                ("v_stride", ctypes.c_int64 * 3), ("o_stride", ctypes.c_int64 * 3)]


class Params(ctypes.Structure):
    _fields_ = [("sort", ctypes.c_int32), ("sort_window", ctypes.c_int64), ("comp", ctypes.c_int32),
                ("beta", ctypes.c_float), ("select", ctypes.c_int32), ("density", ctypes.c_float),
                ("top_p", ctypes.c_float), ("softmax_scale", ctypes.c_float)]


_SEL_FIELDS = ["perm_q", "perm_k", "q_sorted", "k_sorted", "v_sorted", "kv_index", "kv_count", "mask",
               "block_prob", "logits", "threshold", "q_mean", "q_var", "k_mean", "k_var", "q_key", "k_key"]


class SelectionC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in _SEL_FIELDS]


_lib = None


def load() -> ctypes.CDLL:
    """Load libbaatt.so (raises if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BaError(f"{LIB_PATH} is missing: run `python -m paper_2605_19726_b200.build` "
                      "(there is no fallback path)")
    lib = ctypes.CDLL(LIB_PATH)
    P, PA, S = ctypes.POINTER(Problem), ctypes.POINTER(Params), ctypes.POINTER(SelectionC)
    vp, sz, st = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p
    lib.ba_abi_version.restype = ctypes.c_int
    lib.ba_selection_sizes.argtypes = [P, PA, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_int64)]
    lib.ba_selection_sizes.restype = ctypes.c_int
    lib.ba_select_workspace_size.argtypes = [P, PA]
    lib.ba_select_workspace_size.restype = sz
    lib.ba_attention_workspace_size.argtypes = [P, PA]
    lib.ba_attention_workspace_size.restype = sz
    lib.ba_attention_host_workspace_size.argtypes = [P, PA]
    lib.ba_attention_host_workspace_size.restype = sz
    lib.ba_select.argtypes = [P, PA, vp, vp, vp, S, vp, sz, st]
    lib.ba_select.restype = ctypes.c_int
    lib.ba_sparse_attn.argtypes = [P, PA, S, vp, vp, st]
    lib.ba_sparse_attn.restype = ctypes.c_int
    lib.ba_sparse_attn_gather.argtypes = [P, PA, vp, vp, vp, S, vp, vp, st]
    lib.ba_sparse_attn_gather.restype = ctypes.c_int
    lib.ba_block_mass_workspace_size.argtypes = [P, PA]
    lib.ba_block_mass_workspace_size.restype = sz
    lib.ba_block_mass.argtypes = [P, PA, S, vp, vp, vp, sz, st]
    lib.ba_block_mass.restype = ctypes.c_int
    lib.ba_deviation_workspace_size.argtypes = [P, PA]
    lib.ba_deviation_workspace_size.restype = sz
    lib.ba_deviation.argtypes = [P, PA, S, vp, vp, vp, sz, st]
    lib.ba_deviation.restype = ctypes.c_int
    lib.ba_sparse_attn_peers.argtypes = [P, PA, S, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, vp, st]
    lib.ba_sparse_attn_peers.restype = ctypes.c_int
    lib.ba_sparse_attn_multicast.argtypes = [P, PA, S, vp, vp, st]
    lib.ba_sparse_attn_multicast.restype = ctypes.c_int
    lib.ba_sparse_attn_units.argtypes = [P, PA, S, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p),
                                         ctypes.c_int, vp, st]
    lib.ba_sparse_attn_units.restype = ctypes.c_int
    lib.ba_zero_copy_supported.argtypes = [P, PA]
    lib.ba_zero_copy_supported.restype = ctypes.c_int
    lib.ba_attention.argtypes = [P, PA, vp, vp, vp, vp, vp, vp, sz, st]
    lib.ba_attention.restype = ctypes.c_int
    lib.ba_dense_attn.argtypes = [P, PA, vp, vp, vp, vp, vp, st]
    lib.ba_dense_attn.restype = ctypes.c_int
    lib.ba_attention_host.argtypes = [P, PA, vp, vp, vp, vp, vp, sz, st]
    lib.ba_attention_host.restype = ctypes.c_int
    lib.ba_last_launch_count.restype = ctypes.c_int
    lib.ba_check_errors.argtypes = [st]
    lib.ba_check_errors.restype = ctypes.c_int
    lib.ba_attention_kernel_name.argtypes = [P, PA]
    lib.ba_attention_kernel_name.restype = ctypes.c_char_p
    lib.ba_status_string.argtypes = [ctypes.c_int]
    lib.ba_status_string.restype = ctypes.c_char_p
    lib.ba_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


EXPORTED = ["ba_abi_version", "ba_selection_sizes", "ba_select_workspace_size", "ba_attention_workspace_size",
            "ba_select", "ba_sparse_attn", "ba_sparse_attn_gather", "ba_sparse_attn_peers", "ba_sparse_attn_units",
            "ba_sparse_attn_multicast",
            "ba_zero_copy_supported",
            "ba_attention", "ba_dense_attn", "ba_block_mass_workspace_size", "ba_block_mass",
            "ba_deviation_workspace_size", "ba_deviation",
            "ba_attention_host_workspace_size", "ba_attention_host", "ba_last_launch_count", "ba_check_errors",
            "ba_attention_kernel_name",
            "ba_status_string", "ba_last_error"]


def _check(status: int):
    if status != 0:
        lib = load()
        raise BaError(f"{lib.ba_status_string(status).decode()}: {lib.ba_last_error().decode()}")


def attention_kernel_name(q, k, v, block_size=128) -> str:
    prob = make_problem(q, k, v, None, block_size)
    return load().ba_attention_kernel_name(ctypes.byref(prob), ctypes.byref(make_params())).decode()


def zero_copy_supported(q, k, v, block_size=128) -> bool:
    """Q, K and V can all be read through the permutations (no copies)."""
    prob = make_problem(q, k, v, None, block_size)
    return load().ba_zero_copy_supported(ctypes.byref(prob), ctypes.byref(make_params())) == 3


def q_gather_supported(q, k, v, block_size=128) -> bool:
    """Q can be read in place through pi_q (K'/V' copies kept)."""
    prob = make_problem(q, k, v, None, block_size)
    return bool(load().ba_zero_copy_supported(ctypes.byref(prob), ctypes.byref(make_params())) & 1)


def last_launch_count() -> int:
    return load().ba_last_launch_count()


def ba_check_errors(stream=None) -> None:
    """Synchronise the stream and raise the error the attention kernels latched on
    the device, if any (BA_ERR_EMPTY_MASK_ROW for a query block with kv_count < 1,
    S:393; BA_ERR_INVALID_ARGUMENT for a kv_index entry outside [0, N_k))."""
    _check(load().ba_check_errors(_stream(stream)))


def _stream(stream=None) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _strides(t: torch.Tensor):
    assert t.dim() == 4 and t.stride(3) == 1, "tensors must be [b, H, L, d] with unit feature stride"
    return (ctypes.c_int64 * 3)(t.stride(0), t.stride(1), t.stride(2))


def make_problem(q, k, v, out=None, block_size: int = 128) -> Problem:
    dt = {torch.bfloat16: BA_DTYPE_BF16, torch.float32: BA_DTYPE_FP32}.get(q.dtype)
    if dt is None:
        raise BaError(f"dtype {q.dtype} unsupported (bf16, fp32)")
    p = Problem()
    p.batch, p.heads_q, p.len_q, p.head_dim = q.shape[0], q.shape[1], q.shape[2], q.shape[3]
    p.heads_kv, p.len_k = k.shape[1], k.shape[2]
    p.block_size, p.dtype = block_size, dt
    p.q_stride, p.k_stride, p.v_stride = _strides(q), _strides(k), _strides(v)
    if out is not None:
        p.o_stride = _strides(out)
    else:  # contiguous [b, Hq, Lq, d]
        p.o_stride = (ctypes.c_int64 * 3)(q.shape[1] * q.shape[2] * q.shape[3], q.shape[2] * q.shape[3], q.shape[3])
    return p


def make_params(density: float = 0.5, beta: float = 1.0, sort: str = "qk", comp: str = "diag",
                sort_window: int = 0, softmax_scale: float = 0.0, select: int = SELECT_TOPK,
                top_p: float = 0.0) -> Params:
    pa = Params()
    pa.sort, pa.sort_window, pa.comp, pa.beta = SORT[sort], sort_window, COMP[comp], beta
    pa.select, pa.density, pa.top_p, pa.softmax_scale = select, density, top_p, softmax_scale
    return pa


def selection_sizes(prob: Problem, params: Params):
    kap, nq, nk = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(load().ba_selection_sizes(ctypes.byref(prob), ctypes.byref(params), ctypes.byref(kap),
                                     ctypes.byref(nq), ctypes.byref(nk)))
    return kap.value, nq.value, nk.value


def _layout(t: torch.Tensor):
    return (tuple(t.shape), tuple(t.stride()), t.dtype, str(t.device))


def _workspace(nbytes: int, device) -> torch.Tensor:
    # torch's caching allocator returns 512-byte aligned blocks
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


@dataclass
class Selection:
    """Device tensors of a ba_selection (see include/ba_attn.h)."""
    perm_q: torch.Tensor
    perm_k: torch.Tensor
    q_sorted: torch.Tensor
    k_sorted: torch.Tensor
    v_sorted: torch.Tensor
    kv_index: torch.Tensor
    kv_count: torch.Tensor
    kappa: int
    n_q: int
    n_k: int
    mask: Optional[torch.Tensor] = None
    block_prob: Optional[torch.Tensor] = None
    logits: Optional[torch.Tensor] = None
    threshold: Optional[torch.Tensor] = None
    q_mean: Optional[torch.Tensor] = None
    q_var: Optional[torch.Tensor] = None
    k_mean: Optional[torch.Tensor] = None
    k_var: Optional[torch.Tensor] = None
    q_key: Optional[torch.Tensor] = None
    k_key: Optional[torch.Tensor] = None

    def to_c(self) -> SelectionC:
        s = SelectionC()
        for n in _SEL_FIELDS:
            t = getattr(self, n)
            setattr(s, n, None if t is None else t.data_ptr())
        return s


def alloc_selection(q, k, prob: Problem, params: Params, diagnostics: bool = False,
                    zero_copy: bool = False) -> Selection:
    """zero_copy: False = all permuted copies (ba_sparse_attn); "q" = no Q' copy
    (Q read in place through pi_q); True = no copies at all.  The attention half
    runs ba_sparse_attn_gather for "q" / True."""
    kap, nq, nk = selection_sizes(prob, params)
    b, hq, lq, d = q.shape
    hkv, lk = k.shape[1], k.shape[2]
    dev = q.device
    i32 = dict(dtype=torch.int32, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    copy = lambda on, *shape: torch.empty(*shape, dtype=q.dtype, device=dev) if on else None
    kv_copy = zero_copy != True  # noqa: E712  ("q": Q in place, K'/V' copies kept)
    sel = Selection(
        perm_q=torch.empty(b, hq, lq, **i32), perm_k=torch.empty(b, hkv, lk, **i32),
        q_sorted=copy(not zero_copy, b, hq, lq, d), k_sorted=copy(kv_copy, b, hkv, lk, d),
        v_sorted=copy(kv_copy, b, hkv, lk, d),
        kv_index=torch.empty(b, hq, nq, kap, **i32), kv_count=torch.empty(b, hq, nq, **i32),
        kappa=kap, n_q=nq, n_k=nk)
    if diagnostics:
        sel.mask = torch.empty(b, hq, nq, nk, dtype=torch.uint8, device=dev)
        sel.block_prob = torch.empty(b, hq, nq, nk, **f64)
        sel.logits = torch.empty(b, hq, nq, nk, **f64)
        sel.threshold = torch.empty(b, hq, nq, **f64)
        sel.q_mean = torch.empty(b, hq, nq, d, **f64)
        sel.q_var = torch.empty(b, hq, nq, d, **f64)
        sel.k_mean = torch.empty(b, hkv, nk, d, **f64)
        sel.k_var = torch.empty(b, hkv, nk, d, **f64)
        sel.q_key = torch.empty(b, hq, lq, dtype=torch.float32, device=dev)
        sel.k_key = torch.empty(b, hkv, lk, dtype=torch.float32, device=dev)
    return sel


class Context:
    """Holds problem/params structs and a reusable workspace for repeated calls
    (the bench's timed loop calls the library without re-allocating)."""

    def __init__(self, q, k, v, block_size=128, density=0.5, beta=1.0, sort="qk", comp="diag",
                 sort_window=0, softmax_scale=0.0, diagnostics=False, out=None, top_p=None, zero_copy=False):
        """top_p: None = top-kappa (Alg. 1 step 10); a float in (0, 1] = the
        cumulative-mass budget (reading A23), capped at kappa(density).
        zero_copy: False = permuted copies (ba_sparse_attn); "q" = Q read in place
        through pi_q, K'/V' copies (what ba_attention runs); True = no copies, K and
        V gathered through pi_k too (ba_sparse_attn_gather, NEXT-2)."""
        self.zero_copy = zero_copy
        self.prob = make_problem(q, k, v, out, block_size)
        select = SELECT_TOPK if top_p is None else SELECT_TOPP
        self.params = make_params(density, beta, sort, comp, sort_window, softmax_scale, select,
                                  0.0 if top_p is None else top_p)
        lib = load()
        self.ws_select = _workspace(lib.ba_select_workspace_size(ctypes.byref(self.prob), ctypes.byref(self.params)), q.device)
        zc = load().ba_zero_copy_supported(ctypes.byref(self.prob), ctypes.byref(self.params))
        if (zero_copy is True and zc != 3) or (zero_copy == "q" and not zc & 1):
            raise BaError("BA_ERR_UNSUPPORTED: zero-copy attention is not supported for this problem "
                          "(see ba_sparse_attn_gather in include/ba_attn.h)")
        self.sel = alloc_selection(q, k, self.prob, self.params, diagnostics, zero_copy)
        self.sel_c = self.sel.to_c()
        self._layout = tuple(_layout(t) for t in (q, k, v))
        self.qkv = (q, k, v)

    def _check_inputs(self, q, k, v):
        got = tuple(_layout(t) for t in (q, k, v))
        if got != self._layout:
            raise BaError(f"BA_ERR_SHAPE_MISMATCH: q/k/v (shape, stride, dtype, device) {got} differ from the "
                          f"problem this Context was built for {self._layout}")

    def _check_out(self, out, lse=None):
        """out must have the o_stride layout baked into the problem (a mismatch would
        be written with the wrong strides) and the q shape; lse is [b, Hq, Lq] fp32."""
        q = self.qkv[0]
        os = tuple(self.prob.o_stride)
        # strides of size-1 dims are never used for addressing, so they need not match
        same = all(out.shape[i] == 1 or out.stride(i) == os[i] for i in range(3)) if out.dim() == 4 else False
        if tuple(out.shape) != tuple(q.shape) or out.dtype != q.dtype or out.stride(3) != 1 or not same:
            raise BaError(f"BA_ERR_SHAPE_MISMATCH: out {tuple(out.shape)} strides {tuple(out.stride())} do not match "
                          f"the problem's [b, Hq, Lq, d] {tuple(q.shape)} with o_stride {os} (pass out= at construction)")
        if lse is not None and (tuple(lse.shape) != tuple(q.shape[:3]) or lse.dtype != torch.float32
                                or not lse.is_contiguous()):
            raise BaError("BA_ERR_SHAPE_MISMATCH: lse must be a contiguous fp32 [b, Hq, Lq] tensor")

    def _check_sel(self, sel: "Selection"):
        """An injected selection must have this problem's kappa / N_q / N_k: the C side
        strides kv_index rows by kappa(density) of these params."""
        kap, nq, nk = selection_sizes(self.prob, self.params)
        if (sel.kappa, sel.n_q, sel.n_k) != (kap, nq, nk) or tuple(sel.kv_index.shape[2:]) != (nq, kap):
            raise BaError(f"BA_ERR_SHAPE_MISMATCH: selection (kappa, N_q, N_k) = {(sel.kappa, sel.n_q, sel.n_k)} "
                          f"but this Context's params give {(kap, nq, nk)}")

    def select(self, q, k, v, stream=None) -> Selection:
        """Alg. 1 steps 1-10 on (q, k, v), which must have the layout the Context was
        built for; the zero-copy attention then reads these tensors."""
        self._check_inputs(q, k, v)
        _check(load().ba_select(ctypes.byref(self.prob), ctypes.byref(self.params), _ptr(q), _ptr(k), _ptr(v),
                                ctypes.byref(self.sel_c), _ptr(self.ws_select), self.ws_select.numel(),
                                _stream(stream)))
        self.qkv = (q, k, v)
        return self.sel

    def block_mass(self, captured: bool = True, stream=None):
        """NEXT-3: (m_hat [b,Hq,Nq,Nk], captured [b,Hq,Nq]) of the dense softmax in the
        sorted block space for the last selection (ba_block_mass)."""
        lib = load()
        q = self.qkv[0]
        b, hq = q.shape[0], q.shape[1]
        m_hat = torch.empty(b, hq, self.sel.n_q, self.sel.n_k, dtype=torch.float32, device=q.device)
        cap = torch.empty(b, hq, self.sel.n_q, dtype=torch.float32, device=q.device) if captured else None
        ws = _workspace(lib.ba_block_mass_workspace_size(ctypes.byref(self.prob), ctypes.byref(self.params)), q.device)
        _check(lib.ba_block_mass(ctypes.byref(self.prob), ctypes.byref(self.params), ctypes.byref(self.sel_c),
                                 _ptr(m_hat), _ptr(cap), _ptr(ws), ws.numel(), _stream(stream)))
        return m_hat, cap

    def deviation(self, stream=None):
        """NEXT-3: (U, max_dev) [b, Hq, Nq, Nk] fp64 of the last selection (ba_deviation):
        the bound of Eq. logits-bound and the observed max |l_hat - l| per block pair
        (Fig. 2).  Needs a Context built with diagnostics=True."""
        lib = load()
        if self.sel.q_mean is None:
            raise BaError("BA_ERR_INVALID_ARGUMENT: ba_deviation needs the block means (Context(diagnostics=True))")
        q = self.qkv[0]
        b, hq = q.shape[0], q.shape[1]
        U = torch.empty(b, hq, self.sel.n_q, self.sel.n_k, dtype=torch.float64, device=q.device)
        dev = torch.empty_like(U)
        ws = _workspace(lib.ba_deviation_workspace_size(ctypes.byref(self.prob), ctypes.byref(self.params)), q.device)
        _check(lib.ba_deviation(ctypes.byref(self.prob), ctypes.byref(self.params), ctypes.byref(self.sel_c), _ptr(U),
                                _ptr(dev), _ptr(ws), ws.numel(), _stream(stream)))
        return U, dev

    def sparse_attn_peers(self, peer_ptrs, lse=None, stream=None):
        """Fused output collective: store every output row to each of the device
        pointers in peer_ptrs (ba_sparse_attn_peers); strides are those of `out`
        given at construction (contiguous [b, Hq, Lq, d] by default)."""
        arr = (ctypes.c_void_p * len(peer_ptrs))(*[ctypes.c_void_p(int(p)) for p in peer_ptrs])
        _check(load().ba_sparse_attn_peers(ctypes.byref(self.prob), ctypes.byref(self.params), ctypes.byref(self.sel_c),
                                           arr, len(peer_ptrs), _ptr(lse), _stream(stream)))

    def sparse_attn_multicast(self, mc_ptr, lse=None, stream=None):
        """Fused output collective over NVLS: every output row stored once with multimem.st
        to the multicast address mc_ptr (ba_sparse_attn_multicast); strides those of `out`
        given at construction."""
        _check(load().ba_sparse_attn_multicast(ctypes.byref(self.prob), ctypes.byref(self.params),
                                               ctypes.byref(self.sel_c), ctypes.c_void_p(int(mc_ptr)), _ptr(lse),
                                               _stream(stream)))

    def sparse_attn_units(self, unit_begin: int, unit_end: int, outs, lse=None, stream=None):
        """Attention for work units [unit_begin, unit_end) only, u = (b*Hq + h)*Nq + g_q
        (ba_sparse_attn_units): rows stored at their original positions in every
        output of `outs` (tensors or device pointers; strides those of `out` given
        at construction)."""
        for o in outs:
            if isinstance(o, torch.Tensor):
                self._check_out(o)
        if lse is not None and (tuple(lse.shape) != tuple(self.qkv[0].shape[:3]) or lse.dtype != torch.float32
                                or not lse.is_contiguous()):
            raise BaError("BA_ERR_SHAPE_MISMATCH: lse must be a contiguous fp32 [b, Hq, Lq] tensor")
        ptrs = [o.data_ptr() if isinstance(o, torch.Tensor) else int(o) for o in outs]
        arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(p) for p in ptrs])
        _check(load().ba_sparse_attn_units(ctypes.byref(self.prob), ctypes.byref(self.params), ctypes.byref(self.sel_c),
                                           int(unit_begin), int(unit_end), arr, len(ptrs), _ptr(lse), _stream(stream)))

    def sparse_attn(self, out, lse=None, sel: Optional[Selection] = None, stream=None):
        self._check_out(out, lse)
        if sel is not None:
            self._check_sel(sel)
        sc = self.sel_c if sel is None else sel.to_c()
        if self.zero_copy:
            q, k, v = self.qkv
            _check(load().ba_sparse_attn_gather(ctypes.byref(self.prob), ctypes.byref(self.params), _ptr(q), _ptr(k),
                                                _ptr(v), ctypes.byref(sc), _ptr(out), _ptr(lse), _stream(stream)))
        else:
            _check(load().ba_sparse_attn(ctypes.byref(self.prob), ctypes.byref(self.params), ctypes.byref(sc),
                                         _ptr(out), _ptr(lse), _stream(stream)))
        return out


def ba_select(q, k, v, block_size=128, density=0.5, beta=1.0, sort="qk", comp="diag", sort_window=0,
              diagnostics=False, stream=None, top_p=None) -> Selection:
    ctx = Context(q, k, v, block_size, density, beta, sort, comp, sort_window, 0.0, diagnostics, top_p=top_p)
    return ctx.select(q, k, v, stream)


def ba_sparse_attn(q, k, v, sel: Selection, block_size=128, density=None, softmax_scale=0.0,
                   out=None, lse=None, stream=None):
    """Attention half only, with a given (possibly injected) selection.  density:
    None = the selection's own kappa / N_k (the C side strides kv_index rows by
    kappa(density)); an explicit density must give the selection's kappa."""
    if out is None:
        out = torch.empty_like(q)
    prob = make_problem(q, k, v, out, block_size)
    if density is None:
        density = sel.kappa / sel.n_k
    params = make_params(density=density, softmax_scale=softmax_scale)
    kap, nq, nk = selection_sizes(prob, params)
    if (kap, nq, nk) != (sel.kappa, sel.n_q, sel.n_k) or tuple(sel.kv_index.shape[2:]) != (nq, kap):
        raise BaError(f"BA_ERR_SHAPE_MISMATCH: selection (kappa, N_q, N_k) = {(sel.kappa, sel.n_q, sel.n_k)} but "
                      f"density={density}, block_size={block_size} give {(kap, nq, nk)}")
    sc = sel.to_c()
    _check(load().ba_sparse_attn(ctypes.byref(prob), ctypes.byref(params), ctypes.byref(sc), _ptr(out),
                                 _ptr(lse), _stream(stream)))
    return out


def ba_attention(q, k, v, block_size=128, density=0.5, beta=1.0, sort="qk", comp="diag", sort_window=0,
                 softmax_scale=0.0, out=None, lse=None, workspace=None, stream=None, top_p=None):
    if out is None:
        out = torch.empty_like(q)
    prob = make_problem(q, k, v, out, block_size)
    params = make_params(density, beta, sort, comp, sort_window, softmax_scale,
                         SELECT_TOPK if top_p is None else SELECT_TOPP, 0.0 if top_p is None else top_p)
    lib = load()
    need = lib.ba_attention_workspace_size(ctypes.byref(prob), ctypes.byref(params))
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, q.device)
    _check(lib.ba_attention(ctypes.byref(prob), ctypes.byref(params), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                            _ptr(lse), _ptr(workspace), workspace.numel(), _stream(stream)))
    return out


def ba_dense_attn(q, k, v, softmax_scale=0.0, out=None, lse=None, block_size=128, stream=None):
    if out is None:
        out = torch.empty_like(q)
    prob = make_problem(q, k, v, out, block_size)
    params = make_params(density=1.0, sort="none", comp="none", softmax_scale=softmax_scale)
    _check(load().ba_dense_attn(ctypes.byref(prob), ctypes.byref(params), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                _ptr(lse), _stream(stream)))
    return out


def attention_host_workspace_size(q, k, v, block_size=128, density=0.5, beta=1.0, sort="qk", comp="diag",
                                  sort_window=0) -> int:
    prob = make_problem(q, k, v, None, block_size)
    params = make_params(density, beta, sort, comp, sort_window)
    return load().ba_attention_host_workspace_size(ctypes.byref(prob), ctypes.byref(params))


def ba_attention_host(q_host, k_host, v_host, out_host, workspace, block_size=128, density=0.5, beta=1.0,
                      sort="qk", comp="diag", sort_window=0, stream=None):
    """End to end from (pinned) host tensors; enqueues H2D, the path and D2H on
    the stream.  Synchronise the stream before reading out_host."""
    prob = make_problem(q_host, k_host, v_host, out_host, block_size)
    params = make_params(density, beta, sort, comp, sort_window)
    _check(load().ba_attention_host(ctypes.byref(prob), ctypes.byref(params), _ptr(q_host), _ptr(k_host),
                                    _ptr(v_host), _ptr(out_host), _ptr(workspace), workspace.numel(),
                                    _stream(stream)))
    return out_host
