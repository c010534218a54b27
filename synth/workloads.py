"""Seeded synthetic Q/K/V shaped like the paper's workloads.

This module holds NO arithmetic of the method (no norms, sorting, pooling,
scoring, selection or attention).  It is the one module both the CUDA path's
tests/bench and the oracle's tests may use.  The recipe (DESIGN.md "Input
recipe") follows SURVEY.md §8(d1):

  X_i = RoPE(pos_i) · s_i · (z_i + gamma · c_seg(i)) / d^(1/4)

  z ~ N(0, I_d), s ~ LogNormal(0, sigma) (heavy-tailed activations),
  c = segment centres shared by the Q and K of a head (text segments, image
  spans, a smooth spatio-temporal field for video), RoPE as in P:244
  ("RoPE-enhanced queries and keys").  V ~ N(0, I) (reading A19).
  The 1/d^(1/4) factor keeps Q·K/sqrt(d) = O(s_q s_k), i.e. LLM-like logits.

Values are drawn in fp32 with torch generators (CPU or CUDA) and cast to the
target dtype with round-to-nearest-even.  Bit-identity across devices is not
required: the oracle always receives the exact tensors the GPU consumed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

import torch

SEED_BASE = 260519726


@dataclass(frozen=True)
class Workload:
    name: str
    batch: int
    heads_q: int
    heads_kv: int
    seq_len: int
    head_dim: int
    block_size: int
    dtype: str            # "bf16" | "fp32"
    density: float
    kind: str             # "plain" | "text" | "mllm" | "video"
    config_index: int
    sigma_q: float = 1.0
    sigma_k: float = 1.0
    gamma: float = 1.0
    rope_theta: float = 5.0e5

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32


# BASELINE.json "configs" (T, A, C, M, V).
CONFIGS = {
    "T": Workload("tiny", 1, 1, 1, 1024, 64, 64, "fp32", 0.5, "plain", 0,
                  sigma_q=1.0, sigma_k=1.0, gamma=0.0),
    "A": Workload("llada8b_32k", 1, 32, 32, 32768, 128, 128, "bf16", 0.5, "text", 1,
                  sigma_q=0.5, sigma_k=1.0, gamma=1.0),
    "C": Workload("longctx_128k_gqa", 1, 32, 8, 131072, 128, 128, "bf16", 0.5, "text", 2,
                  sigma_q=0.5, sigma_k=1.0, gamma=1.0),
    "M": Workload("mllm_64k", 1, 28, 28, 65536, 128, 64, "bf16", 0.5, "mllm", 3,
                  sigma_q=0.5, sigma_k=1.0, gamma=1.0),
    "V": Workload("video_dit_75600", 1, 24, 24, 75600, 128, 128, "bf16", 0.5, "video", 4,
                  sigma_q=0.5, sigma_k=0.5, gamma=1.0),
}


def _rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    """Rotary embedding on (even, odd) feature pairs; pos [L] float."""
    d = x.shape[-1]
    inv = theta ** (-torch.arange(0, d, 2, device=x.device, dtype=torch.float64) / d)
    ang = (pos.to(torch.float64)[:, None] * inv[None, :]).to(torch.float32)
    c, s = torch.cos(ang), torch.sin(ang)
    xe, xo = x[..., 0::2], x[..., 1::2]
    out = torch.empty_like(x)
    out[..., 0::2] = xe * c - xo * s
    out[..., 1::2] = xe * s + xo * c
    return out


def _rope3d(x: torch.Tensor, f, h, w, theta: float) -> torch.Tensor:
    """3-D RoPE for video: the feature dim is split 44/42/42 (d=128) or in
    thirds rounded to even, each third rotated by one grid coordinate."""
    d = x.shape[-1]
    a = (d // 3 + 1) // 2 * 2 if d != 128 else 44
    b = (d - a) // 2 // 2 * 2
    c = d - a - b
    parts = [x[..., :a], x[..., a:a + b], x[..., a + b:]]
    return torch.cat([_rope(parts[0], f, theta), _rope(parts[1], h, theta),
                      _rope(parts[2], w, theta)], dim=-1)


def _segments_text(L: int, seg: int, device) -> torch.Tensor:
    return torch.arange(L, device=device) // seg


def _gen_head(w: Workload, head: int, centre_head: int, L: int, device,
              which: str) -> torch.Tensor:
    """One head's fp32 [L, d] Q or K (which in {"q","k"}); V handled apart.
    ``centre_head`` (the KV head) seeds the segment centres so that a KV head
    and all q-heads of its GQA group share structure."""
    d = w.head_dim
    g = torch.Generator(device=device)
    g.manual_seed(SEED_BASE + 1000 * w.config_index + 50 + centre_head)
    # centres are shared by Q and K of the head -> drawn first from the same stream
    n_centres = max(1, L // 256 + 64)
    centres = torch.randn(n_centres, d, generator=g, device=device)
    # a per-(head, side) stream for the rest
    g2 = torch.Generator(device=device)
    g2.manual_seed(SEED_BASE + 1000 * w.config_index + head + (500 if which == "k" else 250))
    z = torch.randn(L, d, generator=g2, device=device)
    sigma = w.sigma_q if which == "q" else w.sigma_k
    s = torch.exp(sigma * torch.randn(L, generator=g2, device=device))
    pos = torch.arange(L, device=device, dtype=torch.float32)
    if w.kind in ("plain",):
        x = s[:, None] * (z + w.gamma * centres[_segments_text(L, 1024, device) % n_centres])
        x = x / d ** 0.25
        return x
    if w.kind == "text":
        seg = _segments_text(L, 1024, device) % n_centres
        x = s[:, None] * (z + w.gamma * centres[seg])
        s_sink = torch.ones(L, device=device)
        s_sink[:4] = 8.0  # 4 attention-sink rows
        x = x * s_sink[:, None] / d ** 0.25
        return _rope(x, pos, w.rope_theta)
    if w.kind == "mllm":
        # 24 image spans of 2304 tokens interleaved with text (10240 text tokens at 64K);
        # image tokens: c_img + 0.3 z (low intra-image variance)
        seg = _segments_text(L, 1024, device) % n_centres
        x = s[:, None] * (z + w.gamma * centres[seg])
        n_img, span = 24, 2304
        if L >= n_img * span:
            text_total = L - n_img * span
            gap = text_total // (n_img + 1)
            start = gap
            for i in range(n_img):
                c_img = centres[(i * 7 + 3) % n_centres]
                x[start:start + span] = (c_img[None, :] * 1.5 + 0.3 * z[start:start + span]) * s[start:start + span, None].clamp(max=2.0)
                start += span + gap
        x = x / d ** 0.25
        return _rope(x, pos, w.rope_theta)
    if w.kind == "video":
        # 21 x 45 x 80 latent grid (Wan2.1 720p reading, 75,600 tokens); a smooth
        # field c(f,h,w) = sum_k a_k cos(omega_k . (f,h,w) + phi_k) plus 0.5 z.
        F, H, W = 21, 45, 80
        idx = torch.arange(L, device=device)
        fi = (idx // (H * W)).float()
        hi = ((idx // W) % H).float()
        wi = (idx % W).float()
        gf = torch.Generator(device=device)
        gf.manual_seed(SEED_BASE + 1000 * w.config_index + centre_head + 77)
        field = torch.zeros(L, d, device=device)
        for _ in range(16):
            om = torch.rand(3, generator=gf, device=device) * 0.6
            ph = torch.rand(d, generator=gf, device=device) * 2 * math.pi
            a = torch.randn(d, generator=gf, device=device)
            arg = om[0] * fi + om[1] * hi + om[2] * wi
            field += a[None, :] * torch.cos(arg[:, None] + ph[None, :])
        field = field / 4.0
        x = s[:, None] * (field + 0.5 * z) / d ** 0.25
        return _rope3d(x, fi, hi, wi, 1.0e4)
    raise ValueError(w.kind)


def make_qkv(w: Workload, device="cpu", seq_len: Optional[int] = None,
             heads_q: Optional[int] = None, heads_kv: Optional[int] = None,
             batch: Optional[int] = None, special: bool = True):
    """Return (q, k, v) as contiguous [b, H, L, d] tensors of ``w.dtype`` on
    ``device``.  ``seq_len`` / ``heads_*`` / ``batch`` override the config
    (small parity cases use the same recipe at smaller sizes).  ``special``
    adds the tie / degenerate structure of config T (duplicate rows -> exact
    norm ties; constant runs -> constant blocks)."""
    L = seq_len or w.seq_len
    hq = heads_q or w.heads_q
    hkv = heads_kv or w.heads_kv
    b = batch or w.batch
    d = w.head_dim
    dt = w.torch_dtype
    q = torch.empty(b, hq, L, d, dtype=dt, device=device)
    k = torch.empty(b, hkv, L, d, dtype=dt, device=device)
    v = torch.empty(b, hkv, L, d, dtype=dt, device=device)
    for bi in range(b):
        for h in range(hq):
            wq = w if bi == 0 else w.with_(config_index=w.config_index + 100 * bi)
            q[bi, h] = _gen_head(wq, h, h // (hq // hkv), L, device, "q").to(dt)
        for h in range(hkv):
            wk = w if bi == 0 else w.with_(config_index=w.config_index + 100 * bi)
            k[bi, h] = _gen_head(wk, h, h, L, device, "k").to(dt)
            gv = torch.Generator(device=device)
            gv.manual_seed(SEED_BASE + 1000 * wk.config_index + 900 + h)
            v[bi, h] = torch.randn(L, d, generator=gv, device=device).to(dt)
    if special and w.kind == "plain" and L >= 512:
        # 8 exact duplicate-row pairs (norm ties) and 2 constant runs of B rows
        B = w.block_size
        for i in range(8):
            q[:, :, 100 + 37 * i] = q[:, :, 3 + 11 * i]
            k[:, :, 200 + 29 * i] = k[:, :, 5 + 13 * i]
        q[:, :, 2 * B:3 * B] = q[:, :, 2 * B:2 * B + 1]
        k[:, :, 4 * B:5 * B] = k[:, :, 4 * B:4 * B + 1]
    return q.contiguous(), k.contiguous(), v.contiguous()


def constant_block_qkv(n_blocks: int, B: int, d: int, seed: int = 7, dtype=torch.float64):
    """Q, K with every block of B rows constant (one random row repeated) and
    random V — the special case where pooled logits equal the oracle map
    (P:388).  Returns [L, d] tensors."""
    g = torch.Generator().manual_seed(seed)
    qrows = torch.randn(n_blocks, d, generator=g, dtype=torch.float64)
    krows = torch.randn(n_blocks, d, generator=g, dtype=torch.float64)
    Q = qrows.repeat_interleave(B, dim=0).to(dtype)
    K = krows.repeat_interleave(B, dim=0).to(dtype)
    V = torch.randn(n_blocks * B, d, generator=g, dtype=torch.float64).to(dtype)
    return Q, K, V
