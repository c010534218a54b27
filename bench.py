#!/usr/bin/env python
"""bench.py — BA-Att hot path on B200: block-sparse attention TFLOP/s at 50%
block sparsity (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C|A|V|M|T]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)
    python bench.py --impl reference ...                   (the CPU oracle arm)

A step = one pass of the whole hot path over one batch of synthetic input:
ba_select (Alg. 1 steps 1-10: norm keys, sort, permute + block stats, scores,
top-kappa) + ba_sparse_attn (steps 11-12: tcgen05 block-sparse attention,
un-permute).  `value` = algorithmic FLOPs of the selected block pairs
(4 n_q n_k d per pair, ragged sizes exact) summed over ranks / the max over
ranks of the device time.

Multi-GPU (the north star's 1/2/4/8-GPU head split): `--gpus N`
without a torchrun environment re-launches itself as N ranks
(torch.distributed.run, NCCL, 127.0.0.1).  The default split is head-parallel
STRONG scaling: every rank owns whole GQA groups of the same layer, and the
output is reassembled inside the timed region by one NCCL all-gather (or, with
--fused, by peer stores from the attention epilogue); head counts that do not
divide (M's 28 heads on 8 GPUs) split flattened (head, query-block) units
evenly instead.  `--shard batch` keeps round 1's weak scaling (one batch
element per rank, no collective).  `--dry-run` runs the same launcher,
partition and reassembly on CPU ranks (gloo) with a stand-in kernel — a test
of the plumbing, never a measurement.  Inputs (1.6 GB per step at config C)
are larger than L2 (126 MB).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "block-sparse attn TFLOP/s & speedup vs dense at 50% sparsity, L=32K–128K"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C")
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--top-p", type=float, default=None,
                    help="cumulative-mass budget (BA_SELECT_TOPP, reading A23) capped at --density")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--q-in-place", action="store_true", help="no Q' copy: Q read through pi_q (K'/V' copies)")
    ap.add_argument("--comp", default="diag", choices=["none", "diag", "exact"],
                    help="compensation: diagonal (default), none, or exact covariances (NEXT-4)")
    ap.add_argument("--fidelity", action="store_true",
                    help="NEXT-3: also report the oracle block mass (ba_block_mass): captured mass, Pearson R(m', m_hat)")
    ap.add_argument("--zero-copy", action="store_true",
                    help="NEXT-2: no Q'/K'/V' copies, attention gathers rows through pi (ba_sparse_attn_gather)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / e2e / cpu legs)")
    ap.add_argument("--fused", action="store_true",
                    help="with --shard heads: fuse the output all-gather into the attention epilogue (peer stores "
                         "into symmetric memory, ba_sparse_attn_peers) instead of an NCCL all-gather")
    ap.add_argument("--shard", default=None, choices=["batch", "heads", "units"],
                    help="heads (default): strong scaling, rank r runs a slice of whole GQA groups and O is "
                         "reassembled (NCCL all-gather, or --fused peer stores); falls back to units when the KV "
                         "heads do not divide by the world size; units: strong scaling over evenly split "
                         "(head, q-block) work units (SURVEY 8(e)); batch: weak scaling, rank r runs its own batch "
                         "element, no collective")
    ap.add_argument("--sort", default="qk", choices=["none", "q", "k", "qk"],
                    help="which sides are norm-sorted (P:436-446; ablation P:822-840)")
    ap.add_argument("--beta", type=float, default=1.0, help="compensation weight (P:498)")
    ap.add_argument("--seq-len", type=int, default=None, help="override the config's L")
    ap.add_argument("--block-size", type=int, default=None, choices=[64, 128], help="override the config's B")
    ap.add_argument("--random-lists", action="store_true",
                    help="replace the selection's index lists by uniformly random ones (same kappa): the attention "
                         "kernel on INCOHERENT lists (the pair kernels' union grows from ~1.01 kappa to ~2 kappa)")
    ap.add_argument("--ablation", action="store_true",
                    help="NEXT-3 on synthetic data: per sort mode (none, q, k, qk) the captured dense-softmax mass of "
                         "the selection at 50/70/90%% sparsity (the direction of the Ruler-4K ablation, P:822-840) and "
                         "the per-head Pearson R of U vs the observed max logit deviation (Fig. 2, P:376-405)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU ranks (gloo) with a stand-in for the kernels: checks the launcher, the head / unit "
                         "partition and the output reassembly; prints a JSON line marked dry_run (not a measurement)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"tflops_burst": d.get("bf16_tflops"), "tflops_sustained": d.get("bf16_tflops_sustained"),
                "hbm_gbs": d.get("hbm_gbs"), "source": "measured"}
    return {"tflops_burst": 1590.0, "tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


def workload_desc(w, density, top_p=None, comp="diag", sort="qk", beta=1.0):
    budget = (f"density={density} ({int(round((1 - density) * 100))}% block sparsity)" if top_p is None else
              f"top_p={top_p} capped at density={density} (cumulative-mass budget)")
    return (f"{w.name} (config {w.config_index}): per rank b=1, Hq={w.heads_q}, Hkv={w.heads_kv}, "
            f"L={w.seq_len}, d={w.head_dim}, B={w.block_size}, {budget}, sort={sort}, comp={comp}, beta={beta:g}")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-lms", "200"],
                                     stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
                except ValueError:
                    pass
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        sm = sorted(r[0] for r in rows)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------------- FLOPs
def sparse_flops_from_index(kv_index, kv_count, lq, lk, B, d, units=None):
    """Sum over selected pairs of 4 n_q n_k d (QK^T + PV), ragged sizes exact;
    `units` = (u0, u1) restricts it to the work units u = (b*H + h)*N_q + g_q."""
    import torch
    nq = kv_index.shape[2]
    nk_tot = (lk + B - 1) // B
    last_k = lk - (nk_tot - 1) * B
    nq_rows = torch.full((nq,), B, dtype=torch.float64, device=kv_index.device)
    nq_rows[-1] = lq - (nq - 1) * B
    kap = kv_index.shape[3]
    valid = torch.arange(kap, device=kv_index.device)[None, None, None, :] < kv_count[..., None]
    nk_sizes = torch.where(kv_index == nk_tot - 1, float(last_k), float(B)).double() * valid
    per_row = nk_sizes.sum(-1)  # [b, h, nq]
    per_unit = (per_row * nq_rows[None, None, :]).flatten()
    if units is not None:
        per_unit = per_unit[units[0]:units[1]]
    return float(per_unit.sum().item()) * 4.0 * d


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return len(os.sched_getaffinity(0))


# --------------------------------------------------------------------------- oracle sample
def oracle_sample(w, q, k, v, density, n_blocks, seed=0, sort="qk", beta=1.0, comp="diag"):
    """Run the fp64 oracle on a bounded sample of the workload: the full
    selection (Alg. 1 steps 1-10) of one q-head and block-sparse attention
    for `n_blocks` of its query blocks.  Returns (flops, seconds, desc)."""
    import numpy as np
    import oracle as O
    t0 = time.perf_counter()
    sel = O.select_head(q, k, w.block_size, density, beta, {"none": O.SORT_NONE, "q": O.SORT_Q, "k": O.SORT_K,
                                                             "qk": O.SORT_QK}[sort],
                        {"none": O.COMP_NONE, "diag": O.COMP_DIAG, "exact": O.COMP_EXACT}[comp])
    t_sel = time.perf_counter() - t0
    Qs = O.apply_permutation(q, sel.perm_q)
    Ks = O.apply_permutation(k, sel.perm_k)
    Vs = O.apply_permutation(v, sel.perm_k)
    nq = sel.kv_index.shape[0]
    rng = np.random.default_rng(seed)
    blocks = sorted(set([0, nq - 1] + list(rng.choice(nq, size=min(nq, n_blocks), replace=False))))[:n_blocks]
    t1 = time.perf_counter()
    O.block_sparse_attention_head(Qs, Ks, Vs, sel.kv_index, w.block_size, 1.0 / math.sqrt(w.head_dim), blocks)
    t_attn = time.perf_counter() - t1
    # FLOPs of the sampled query blocks (ragged exact)
    L = q.shape[0]
    fl = 0
    for g in blocks:
        nqr = min(w.block_size, L - g * w.block_size)
        for j in sel.kv_index[g]:
            nkr = min(w.block_size, k.shape[0] - int(j) * w.block_size)
            fl += 4 * nqr * nkr * w.head_dim
    # selection pro-rated to the sampled share of the head's query blocks
    secs = t_attn + t_sel * len(blocks) / nq
    desc = (f"oracle (fp64 NumPy) on 1 q-head of the workload: full selection ({t_sel:.2f}s, pro-rated "
            f"{len(blocks)}/{nq}) + block-sparse attention of {len(blocks)} query blocks ({t_attn:.2f}s)")
    return fl, secs, desc


def oracle_dense_sample(w, q, k, v, n_rows):
    """The oracle's dense attention for the first `n_rows` query rows
    of one head against every key, timed as the CPU dense reference (SURVEY
    8(d4)).  Returns (flops, seconds)."""
    import oracle as O
    t0 = time.perf_counter()
    O.dense_attention(q[:n_rows], k, v, 1.0 / math.sqrt(w.head_dim), row_block=128)
    return 4.0 * n_rows * k.shape[0] * w.head_dim, time.perf_counter() - t0


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # under torchrun only rank 0 runs the CPU oracle arm
    from synth import make_qkv
    w = make_workload(args)
    density = args.density if args.density is not None else w.density
    # one head of the workload, generated on the host (same recipe as the GPU arm)
    q, k, v = make_qkv(w, device="cpu", heads_q=1, heads_kv=1)
    qn, kn, vn = q[0, 0].float().numpy(), k[0, 0].float().numpy(), v[0, 0].float().numpy()
    n_blocks = 8 if w.seq_len >= 65536 else 16
    for _ in range(args.warmup):
        oracle_sample(w, qn, kn, vn, density, 2, sort=args.sort, beta=args.beta, comp=args.comp)
    tot_fl, tot_s, desc = 0, 0.0, ""
    for s in range(args.steps):
        fl, secs, desc = oracle_sample(w, qn, kn, vn, density, n_blocks, seed=s, sort=args.sort, beta=args.beta,
                                       comp=args.comp)
        tot_fl += fl
        tot_s += secs
    value = tot_fl / tot_s / 1e12
    cores = cpu_cores()
    line = {"impl": "reference", "schema": "ba-bench-line/2", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if args.shard == "batch" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(w, density, args.top_p, args.comp, args.sort, args.beta),
                       "global_batch": args.gpus if args.shard == "batch" else 1, "seq_len": w.seq_len,
                       "parallelism": "oracle on the host cores of rank 0 (bounded sample of the same layer)"},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
def make_workload(args):
    from synth import CONFIGS
    w = CONFIGS[args.config]
    if args.seq_len is not None:
        w = w.with_(seq_len=args.seq_len)
    if args.block_size is not None:
        w = w.with_(block_size=args.block_size)
    return w


def launch_ranks(args) -> int:
    """`--gpus N` outside torchrun: re-launch this script as N ranks, one per GPU
    (torch.distributed.run on 127.0.0.1), exactly as the driver's multi-GPU launch."""
    import socket
    if not args.dry_run:
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus}: only {n} GPU(s) visible\n")
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def random_lists(kv_index, n_k, seed=0):
    """Uniformly random ascending index lists with the selection's kappa (incoherent
    lists: adjacent query blocks share ~kappa/N_k of their blocks)."""
    import torch
    b, h, nq, kap = kv_index.shape
    g = torch.Generator(device=kv_index.device).manual_seed(seed)
    r = torch.rand(b * h * nq, n_k, generator=g, device=kv_index.device)
    idx = r.argsort(dim=-1)[:, :kap].sort(dim=-1).values
    return idx.to(torch.int32).reshape(b, h, nq, kap).contiguous()


def union_ratio(kv_index, n_k):
    """Mean |list(2p) u list(2p+1)| / kappa over the pair kernels' query-block pairs."""
    import torch
    b, h, nq, kap = kv_index.shape
    m = torch.zeros(b * h * nq, n_k, dtype=torch.bool, device=kv_index.device)
    m.scatter_(1, kv_index.reshape(-1, kap).long(), True)
    m = m.reshape(b * h, nq, n_k)
    npair = nq // 2
    u = (m[:, 0:2 * npair:2] | m[:, 1:2 * npair:2]).sum(-1).double()
    return float(u.mean() / kap) if npair else 1.0


def run_ours(args):
    import torch
    import torch.distributed as dist
    from synth import make_qkv
    from paper_2605_19726_b200.dist import (even_split, gather_heads, gather_units, head_range, max_over_ranks,
                                            sum_over_ranks, unit_heads, unit_range)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dry = args.dry_run
    if dry:  # plumbing check on CPU ranks: no kernels, no timing claims
        dev = torch.device("cpu")
        if world > 1:
            dist.init_process_group("gloo")
        ba = None
    else:
        if not torch.cuda.is_available():
            raise SystemExit("bench.py needs a CUDA device (no CPU fallback); --dry-run checks the plumbing on CPU")
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        if world > 1 or (args.fused and "MASTER_ADDR" in os.environ):  # symmetric memory needs a process group
            dist.init_process_group("nccl", device_id=dev)
        import paper_2605_19726_b200.baatt as ba
        ba.load()
    w = make_workload(args)
    density = args.density if args.density is not None else w.density
    shard = args.shard or "heads"
    heads = shard in ("heads", "units")
    fused = None
    units = None      # (u0, u1) relative to this rank's head slice in the (head, q-block) unit split
    out_local = None  # unit split: zero-filled full-size O holding this rank's rows only
    out_full = None   # the reassembled O
    B = w.block_size
    nq_full = (w.seq_len + B - 1) // B
    if heads:
        # strong scaling: every rank builds the same layer and keeps whole GQA groups
        if shard == "heads" and even_split(w.heads_q, w.heads_kv, world):
            q0, q1, k0, k1 = head_range(w.heads_q, w.heads_kv, world, rank)
        else:
            # SURVEY §8(e) fallback (e.g. M's 28 heads on 8 GPUs): split the flattened (head, q-block)
            # units evenly; a rank selects over the heads its units touch (whole GQA groups)
            u0, u1 = unit_range(w.heads_q, nq_full, world, rank)
            q0, q1, k0, k1 = unit_heads(u0, u1, nq_full, w.heads_q, w.heads_kv)
            units = (u0 - q0 * nq_full, u1 - q0 * nq_full)
        if dry:
            q = torch.zeros(1, q1 - q0, w.seq_len, w.head_dim, dtype=w.torch_dtype)
            k = v = None
        else:
            q, k, v = make_qkv(w, device=dev)
            q, k, v = q[:, q0:q1].contiguous(), k[:, k0:k1].contiguous(), v[:, k0:k1].contiguous()
    else:
        # weak scaling: rank r processes batch element r (its own seeded inputs)
        q0, q1 = 0, w.heads_q
        if dry:
            q = torch.zeros(1, w.heads_q, w.seq_len, w.head_dim, dtype=w.torch_dtype)
            k = v = None
        else:
            wr = w.with_(config_index=w.config_index + 100 * rank)
            q, k, v = make_qkv(wr, device=dev)
    full_shape = (q.shape[0], w.heads_q, q.shape[2], q.shape[3])
    if not dry:
        torch.cuda.synchronize()
    zero_copy = False
    if not dry:
        # the product path (what ba_attention runs) materialises Q'/K'/V'; --zero-copy measures NEXT-2
        # (no copies), --q-in-place only Q read through pi_q
        zero_copy = (True if args.zero_copy and ba.zero_copy_supported(q, k, v, B)
                     else "q" if args.q_in_place and ba.q_gather_supported(q, k, v, B) else False)
    if heads and args.fused and not dry:
        # the output collective fused into the attention epilogue: full O in symmetric memory on
        # every rank, each rank's kernel stores its heads' rows into all copies (NVLink peer stores)
        from paper_2605_19726_b200.dist import FusedHeadGather
        fused = FusedHeadGather(full_shape, q.dtype, dev, q0)
        out = fused.full[:, q0:q1]
        out_full = fused.full
    elif units is not None:
        out_local = torch.zeros(full_shape, dtype=q.dtype, device=dev)
        out = out_local[:, q0:q1]
        out_full = torch.empty_like(out_local) if world > 1 else out_local
    else:
        out = torch.empty_like(q)
    if args.random_lists and (units is not None or fused is not None):
        raise SystemExit("--random-lists runs on the plain ba_sparse_attn path (not with units / --fused)")
    ctx = None
    if not dry:
        ctx = ba.Context(q, k, v, B, density, args.beta, args.sort, args.comp, top_p=args.top_p,
                         zero_copy=zero_copy, out=out)
    stream = torch.cuda.current_stream() if not dry else None
    run_sel = None  # the selection the attention reads (--random-lists: same copies, random index lists)

    def select():
        if dry:
            return 0
        ctx.select(q, k, v)
        return ba.last_launch_count()

    def attn():
        if dry:  # stand-in for the kernels: row t of head h (global) = h*nq + t//B, at the rank's rows only
            if units is not None:
                for u in range(units[0], units[1]):
                    h, g = divmod(u, nq_full)
                    out[0, h, g * B:(g + 1) * B] = (q0 + h) * nq_full + g
            else:
                hh = torch.arange(q0, q1, dtype=torch.float32)[:, None]
                tt = torch.div(torch.arange(w.seq_len), B, rounding_mode="floor").float()[None, :]
                out[0] = (hh * nq_full + tt)[..., None].to(out.dtype)
            return 0
        if units is not None:
            ctx.sparse_attn_units(units[0], units[1], fused.peer_ptrs if fused is not None else [out])
        elif fused is not None:
            if fused.mc_ptr:
                ctx.sparse_attn_multicast(fused.mc_ptr)  # NVLS: one multimem.st per row reaches every rank
            else:
                ctx.sparse_attn_peers(fused.peer_ptrs)
        else:
            ctx.sparse_attn(out, sel=run_sel)
        return ba.last_launch_count()

    def gather():
        """The path's only collective: reassemble O on every rank (strong scaling)."""
        nonlocal out_full
        if world == 1:
            return
        if fused is not None:
            fused.barrier()
        elif units is not None:
            gather_units(out_local, out_full)  # every row has one writer: out-of-place SUM reduction
        elif heads:
            out_full = gather_heads(out, w.heads_q)  # NCCL all-gather over NVLink / NVSwitch

    def step():
        n = select()
        n += attn()
        gather()
        return n

    launches = step()
    if args.random_lists:
        import dataclasses
        run_sel = dataclasses.replace(ctx.sel, kv_index=random_lists(ctx.sel.kv_index, ctx.sel.n_k))
    for _ in range(max(args.warmup, 1)):
        launches = step()
    if not dry:
        torch.cuda.synchronize()
    dry_check = None
    if dry:
        # every rank must now hold the whole layer's O, exactly as one rank would produce it
        if heads:
            res = out_full if (world > 1 or units is not None) else out
            hh = torch.arange(w.heads_q, dtype=torch.float32)[:, None]
            tt = torch.div(torch.arange(w.seq_len), B, rounding_mode="floor").float()[None, :]
            exp = (hh * nq_full + tt)[..., None].expand(-1, -1, w.head_dim).to(q.dtype)
            ok = res is not None and tuple(res.shape[1:]) == tuple(exp.shape) and torch.equal(res[0], exp)
        else:
            ok = True
        ok_all = sum_over_ranks(1.0 if ok else 0.0, dev) == world
        dry_check = "reassembled O equals the 1-rank layout on every rank" if ok_all else "MISMATCH"
    if dry:
        flops_per_step = 0.0
    else:
        kvi = run_sel.kv_index if run_sel is not None else ctx.sel.kv_index
        flops_per_step = sparse_flops_from_index(kvi, ctx.sel.kv_count, q.shape[2], k.shape[2], B, w.head_dim, units)
    sampler = ClockSampler(local) if not args.profile and not dry else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if not dry:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    if not dry:
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
    wall0 = time.perf_counter()
    for i in range(args.steps):
        if not dry:
            ev[i][0].record(stream)
        select()
        if not dry:
            ev[i][1].record(stream)
        attn()
        if not dry:
            ev[i][2].record(stream)
        gather()
    if not dry:
        t_end.record(stream)
        torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    if dry:
        total_ms, sel_each, attn_each = wall * 1e3, [0.0] * args.steps, [0.0] * args.steps
    else:
        total_ms = t_start.elapsed_time(t_end)
        sel_each = [e[0].elapsed_time(e[1]) for e in ev]
        attn_each = [e[1].elapsed_time(e[2]) for e in ev]
    sel_ms = sum(sel_each) / args.steps
    attn_ms = sum(attn_each) / args.steps

    def pcts(xs):  # per-stage distribution over the timed steps (median, p10, p90)
        ys = sorted(xs)
        q_ = lambda f: ys[min(len(ys) - 1, max(0, int(round(f * (len(ys) - 1)))))]
        return {"median": q_(0.5), "p10": q_(0.1), "p90": q_(0.9)}
    ms_per_step = max_over_ranks(total_ms / args.steps, dev)
    sel_ms_max = max_over_ranks(sel_ms, dev)
    attn_ms_max = max_over_ranks(attn_ms, dev)
    flops_all = sum_over_ranks(flops_per_step, dev)
    value = flops_all / (ms_per_step * 1e-3) / 1e12 if ms_per_step > 0 else 0.0
    peaks = load_peaks()
    attn_tflops = flops_per_step / (attn_ms * 1e-3) / 1e12 if attn_ms > 0 else 0.0

    res = {}
    if not args.no_dense and not args.profile and not dry and world == 1:
        # dense references on the same inputs: our tcgen05 kernel with every block
        # (the 1/rho ceiling) and torch SDPA (cuDNN / flash) as an external check
        dn_out = torch.empty_like(q)
        for _ in range(2):
            ba.ba_dense_attn(q, k, v, out=dn_out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = 3
        e0.record(stream)
        for _ in range(nrep):
            ba.ba_dense_attn(q, k, v, out=dn_out)
        e1.record(stream)
        torch.cuda.synchronize()
        dense_ms = e0.elapsed_time(e1) / nrep
        dense_flops = 4.0 * q.shape[0] * q.shape[1] * q.shape[2] * k.shape[2] * q.shape[3]
        res["dense_ms"] = dense_ms
        res["dense_tflops"] = dense_flops / (dense_ms * 1e-3) / 1e12
        res["speedup_vs_dense"] = dense_ms / (total_ms / args.steps)
        try:
            import torch.nn.functional as F
            for _ in range(2):
                F.scaled_dot_product_attention(q, k, v, enable_gqa=q.shape[1] != k.shape[1])
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(nrep):
                F.scaled_dot_product_attention(q, k, v, enable_gqa=q.shape[1] != k.shape[1])
            e1.record(stream)
            torch.cuda.synchronize()
            res["sdpa_ms"] = e0.elapsed_time(e1) / nrep
            res["sdpa_tflops"] = dense_flops / (res["sdpa_ms"] * 1e-3) / 1e12
            res["speedup_vs_sdpa"] = res["sdpa_ms"] / (total_ms / args.steps)
        except Exception as ex:  # SDPA is context only
            res["sdpa_error"] = str(ex)[:120]
        del dn_out

    e2e = None
    if not args.no_e2e and not args.profile and not dry and not args.random_lists:
        qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
        oh = torch.empty(q.shape, dtype=q.dtype).pin_memory()
        n_e2e = max(2, min(args.steps, 5))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world == 1 and units is None:
            # one GPU: the library's end-to-end host API (chunked, copies overlapped with compute)
            ws = torch.empty(ba.attention_host_workspace_size(qh, kh, vh, B, density, args.beta, args.sort,
                                                              args.comp), dtype=torch.uint8, device=dev)
            run = lambda: ba.ba_attention_host(qh, kh, vh, oh, ws, B, density, args.beta, args.sort, args.comp)
            api = "ba_attention_host (pinned host q/k/v -> H2D -> select + sparse attn -> D2H out)"
        else:
            # N ranks: each rank copies its slice in (H2D), runs ba_select + attention, the output is
            # reassembled by the collective (inside the timed region), and the rank's slice is read back
            def run():
                q.copy_(qh, non_blocking=True)
                k.copy_(kh, non_blocking=True)
                v.copy_(vh, non_blocking=True)
                step()
                oh.copy_(out, non_blocking=True)
            api = ("per rank: H2D of its q/k/v slice (pinned) -> ba_select + ba_sparse_attn -> output collective "
                   "-> D2H of its output slice")
        run()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(n_e2e):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / n_e2e, dev)
        h2d = sum_over_ranks(float((qh.numel() + kh.numel() + vh.numel()) * qh.element_size()), dev)
        d2h = sum_over_ranks(float(oh.numel() * oh.element_size()), dev)
        e2e = {"value": flops_all / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "api": api}
        del qh, kh, vh, oh

    fidelity = None
    if args.fidelity and B == 128 and not args.profile and not dry:
        fidelity = run_fidelity(args, ba, q, k, v, B, density, stream)
    ablation = None
    if args.ablation and B == 128 and not args.profile and not dry:
        ablation = run_ablation(args, ba, q, k, v, B)

    cpu = None
    if rank == 0 and not args.no_cpu and not args.profile and world == 1 and not dry:
        hsel = 0
        qn = q[0, hsel].float().cpu().numpy()
        kn = k[0, hsel * k.shape[1] // q.shape[1]].float().cpu().numpy()
        vn = v[0, hsel * k.shape[1] // q.shape[1]].float().cpu().numpy()
        n_blocks = 8 if w.seq_len >= 65536 else 16
        fl, secs, desc = oracle_sample(w, qn, kn, vn, density, n_blocks, sort=args.sort, beta=args.beta,
                                       comp=args.comp)
        cpu = {"value": fl / secs / 1e12, "unit": "TFLOP/s", "cores": cpu_cores(), "kind": "oracle", "sample": desc}
        n_rows = min(qn.shape[0], 4 * B)
        dfl, dsecs = oracle_dense_sample(w, qn, kn, vn, n_rows)
        cpu["dense"] = {"value": dfl / dsecs / 1e12, "unit": "TFLOP/s",
                        "sample": f"oracle dense attention of {n_rows} query rows of 1 head against all {kn.shape[0]} "
                                  f"keys ({dsecs:.2f}s)",
                        "ms_per_step_extrapolated": dsecs * (q.shape[1] * q.shape[2] / n_rows) * 1e3}

    traffic = None
    tp = os.path.join(ROOT, "profiles", "attn_traffic.json")
    if os.path.exists(tp) and not dry:
        try:
            with open(tp) as f:
                tj = json.load(f)
            kname = ba.attention_kernel_name(q, k, v, B)
            for e in tj.get("entries", [tj]):
                if (e.get("config") == args.config and e.get("kernel") == kname and args.density is None
                        and args.top_p is None and not args.random_lists and world == 1):
                    traffic = e.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank == 0:
        tokens = q.shape[2] * (1 if heads else world)
        if units is not None:
            par = (f"unit-parallel x{world} ((head, q-block) units split evenly, "
                   + ("O by peer stores in the attention epilogue)" if fused is not None
                      else "NCCL out-of-place SUM reduction of the zero-filled O)"))
        elif heads:
            par = (f"head-parallel x{world} (whole GQA groups per rank, "
                   + (("O gathered by NVLS multimem.st in the attention epilogue)" if fused.mc_ptr else
                       "O gathered by peer stores in the attention epilogue)") if fused is not None
                      else "NCCL all-gather of O)" if world > 1 else "one rank holds every head)"))
        else:
            par = f"batch-parallel x{world} (weak scaling, no data-path collective)"
        kernel = ba.attention_kernel_name(q, k, v, B) if not dry else "dry-run stand-in"
        line = {
            "schema": "ba-bench-line/2", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if heads else "weak",
            "vs_baseline": None, "dtype": "bf16" if w.dtype == "bf16" else "fp32", "data": "synthetic",
            "config": {"workload": workload_desc(w, density, args.top_p, args.comp, args.sort, args.beta),
                       "global_batch": 1 if heads else world, "seq_len": w.seq_len, "parallelism": par,
                       "heads_per_rank": [q0, q1],
                       "l2": "inputs larger than L2 (q+k+v = %.2f GB per step)" %
                             ((q.numel() * 3 if dry else q.numel() + k.numel() + v.numel()) * 2 / 1e9),
                       "zero_copy": zero_copy, "index_lists": "random (--random-lists)" if args.random_lists
                       else "selected"},
            "roofline": {"bound": "tensor", "kernel": kernel, "achieved": attn_tflops,
                         "peak": peaks["tflops_sustained"], "unit": "TFLOP/s",
                         "frac": attn_tflops / peaks["tflops_sustained"],
                         "peak_kind": f"{peaks['source']} bf16 sustained (kernel timed inside a long step)",
                         "frac_of_burst": attn_tflops / peaks["tflops_burst"],
                         "flops_per_launch": flops_per_step, "ms_per_launch": attn_ms, "traffic": traffic},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clocks,
            "select_ms": sel_ms, "attn_ms": attn_ms, "select_share": sel_ms / (sel_ms + attn_ms) if attn_ms else 0.0,
            "select_ms_max_rank": sel_ms_max, "attn_ms_max_rank": attn_ms_max,
            "stage_ms": {"ba_select": pcts(sel_each), "ba_sparse_attn": pcts(attn_each)},
            "tokens_per_s": tokens / (ms_per_step * 1e-3),
            "flops_per_step_per_rank": flops_per_step,
        }
        if args.random_lists and not dry:
            line["union_ratio"] = {"random": union_ratio(run_sel.kv_index, ctx.sel.n_k),
                                   "selected": union_ratio(ctx.sel.kv_index, ctx.sel.n_k)}
        if dry:
            line["dry_run"] = dry_check
            line["value"] = None
        if fidelity:
            line["fidelity"] = fidelity
        if ablation:
            line["ablation"] = ablation
        line.update(res)
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def run_fidelity(args, ba, q, k, v, B, density, stream):
    """NEXT-3 diagnostics on the GPU: m_hat (Eq. oracle-dist) of the dense softmax in the sorted
    block space vs the selection's m': captured mass and Pearson R per head."""
    import torch
    fctx = ba.Context(q, k, v, B, density, args.beta, args.sort, args.comp, top_p=args.top_p, diagnostics=True)
    fsel = fctx.select(q, k, v)
    fctx.block_mass()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    m_hat, cap = fctx.block_mass()
    e1.record(stream)
    torch.cuda.synchronize()
    mp = fsel.block_prob.float()
    x = mp.flatten(2) - mp.flatten(2).mean(-1, keepdim=True)
    y = m_hat.flatten(2) - m_hat.flatten(2).mean(-1, keepdim=True)
    r = (x * y).sum(-1) / (x.norm(dim=-1) * y.norm(dim=-1))
    return {"block_mass_ms": e0.elapsed_time(e1), "captured_mass_mean": float(cap.mean()),
            "captured_mass_min_row": float(cap.min()), "pearson_r_mprime_mhat_mean": float(r.mean()),
            "pearson_r_min_head": float(r.min()), "random_selection_mass": fsel.kappa / fsel.n_k,
            "what": "m_hat = dense softmax mass per (sorted) block pair (ba_block_mass); captured = "
                    "sum of m_hat over the selected blocks per query block"}


def pearson_rows(x, y):
    """Pearson R of x and y along the last axis (per head)."""
    x = x - x.mean(-1, keepdim=True)
    y = y - y.mean(-1, keepdim=True)
    return (x * y).sum(-1) / (x.norm(dim=-1) * y.norm(dim=-1))


def run_ablation(args, ba, q, k, v, B):
    """NEXT-3 on the GPU (reporting only; every quantity comes from library kernels):
    per sort mode, m_hat (Eq. oracle-dist, ba_block_mass) in that mode's block space and
    the captured mass sum_{M=1} m_hat of the top-kappa selection at 50/70/90% sparsity
    (the Ruler-4K ablation's direction); U and the observed max logit
    deviation (ba_deviation) with their per-head Pearson R (Fig. 2 blue = unsorted,
    red = sorted)."""
    import torch
    t0 = time.perf_counter()
    out = {}
    for sort in ("none", "q", "k", "qk"):
        ctx = ba.Context(q, k, v, B, 0.5, args.beta, sort, args.comp, diagnostics=True)
        ctx.select(q, k, v)
        m_hat, _ = ctx.block_mass(captured=False)
        U, dev = ctx.deviation()
        r = pearson_rows(U.flatten(2), dev.flatten(2))[0]
        row = {"pearson_r_U_maxdev_mean": float(r.mean()), "pearson_r_U_maxdev_min_head": float(r.min()),
               "U_mean": float(U.mean()), "max_dev_mean": float(dev.mean())}
        for dens in (0.5, 0.3, 0.1):
            c2 = ba.Context(q, k, v, B, dens, args.beta, sort, args.comp)
            sel = c2.select(q, k, v)
            cap = m_hat.gather(-1, sel.kv_index.long()).sum(-1)
            row[f"captured_mass_sparsity_{int(round((1 - dens) * 100))}"] = float(cap.mean())
            del c2, sel
        out[sort] = row
        del ctx, m_hat, U, dev
    torch.cuda.synchronize()
    out["what"] = ("captured = mean over query blocks of the dense softmax mass (m_hat, Eq. oracle-dist) the "
                   "top-kappa selection keeps; pearson = per-head R of U (Eq. logits-bound) vs max |l_hat - l| "
                   "over the block pairs; synthetic workload, not the paper's data")
    out["seconds"] = time.perf_counter() - t0
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
