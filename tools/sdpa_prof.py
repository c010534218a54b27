"""Profiling driver (ncu only): cuDNN SDPA and our dense kernel on the same
dense problem (config A shapes, 8 heads), for a side-by-side ncu capture."""
import sys, torch
sys.path.insert(0, '.')
from synth import CONFIGS, make_qkv
import torch.nn.functional as F
import paper_2605_19726_b200.baatt as ba
w = CONFIGS["A"]
q, k, v = make_qkv(w, device="cuda", heads_q=8, heads_kv=8)
for _ in range(2):
    o = F.scaled_dot_product_attention(q, k, v)
    o2 = ba.ba_dense_attn(q, k, v)
torch.cuda.synchronize()
print("ok")
