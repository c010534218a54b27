"""CPU-side checks of the boundary (no compute calls; runs with -m "not gpu").

 - libbaatt.so loads and exports every function include/ba_attn.h declares;
 - the ctypes structs match the C layout (field offsets parsed from the header
   are not available without a compiler, so sizes are checked through a tiny
   C program when gcc is present);
 - synchronous validation returns the documented error codes;
 - the product package never imports the oracle and has no CPU fallback.
"""
import ctypes
import os
import re
import subprocess
import sys
import tempfile

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ba_attn.h")


@pytest.fixture(scope="module")
def ba():
    import paper_2605_19726_b200.baatt as ba
    return ba


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ba_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(ba):
    lib = ba.load()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), f"libbaatt.so does not export {n}"
    assert set(names) == set(ba.EXPORTED)
    assert lib.ba_abi_version() == 1


def test_struct_layout_matches_header(ba, tmp_path):
    code = r"""
#include <stdio.h>
#include <stddef.h>
#include "ba_attn.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(ba_problem), sizeof(ba_params), sizeof(ba_selection),
         offsetof(ba_problem, q_stride), offsetof(ba_problem, o_stride), offsetof(ba_params, density),
         offsetof(ba_selection, k_key));
  return 0;
}
"""
    c = tmp_path / "t.c"
    c.write_text(code)
    exe = tmp_path / "t"
    r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", str(c), "-o", str(exe)],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("gcc / cuda headers unavailable: " + r.stderr[-200:])
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    expect = [ctypes.sizeof(ba.Problem), ctypes.sizeof(ba.Params), ctypes.sizeof(ba.SelectionC),
              ba.Problem.q_stride.offset, ba.Problem.o_stride.offset, ba.Params.density.offset,
              ba.SelectionC.k_key.offset]
    assert vals == expect


def _meta(b, hq, hkv, L, d, dtype=torch.bfloat16):
    q = torch.empty(b, hq, L, d, dtype=dtype, device="meta")
    k = torch.empty(b, hkv, L, d, dtype=dtype, device="meta")
    return q, k, k


def test_sizes_and_kappa(ba):
    q, k, v = _meta(1, 32, 8, 131072, 128)
    p = ba.make_problem(q, k, v)
    assert ba.selection_sizes(p, ba.make_params(0.5)) == (512, 1024, 1024)
    assert ba.selection_sizes(p, ba.make_params(0.25)) == (256, 1024, 1024)
    q, k, v = _meta(1, 24, 24, 75600, 128)
    p = ba.make_problem(q, k, v)
    assert ba.selection_sizes(p, ba.make_params(0.5)) == (296, 591, 591)
    assert ba.selection_sizes(p, ba.make_params(0.4)) == (236, 591, 591)
    q, k, v = _meta(1, 28, 28, 65536, 128)
    p = ba.make_problem(q, k, v, block_size=64)
    assert ba.selection_sizes(p, ba.make_params(0.5)) == (512, 1024, 1024)
    lib = ba.load()
    assert lib.ba_select_workspace_size(ctypes.byref(p), ctypes.byref(ba.make_params())) > 0
    assert lib.ba_attention_workspace_size(ctypes.byref(p), ctypes.byref(ba.make_params())) > \
        lib.ba_select_workspace_size(ctypes.byref(p), ctypes.byref(ba.make_params()))


@pytest.mark.parametrize("mutate,code", [
    (lambda p, pa: setattr(pa, "density", 0.0), "INVALID_ARGUMENT"),
    (lambda p, pa: setattr(pa, "density", 1.5), "INVALID_ARGUMENT"),
    (lambda p, pa: setattr(p, "heads_kv", 3), "SHAPE_MISMATCH"),
    (lambda p, pa: setattr(p, "head_dim", 96), "UNSUPPORTED"),
    (lambda p, pa: setattr(p, "block_size", 32), "UNSUPPORTED"),
    (lambda p, pa: setattr(p, "len_q", 0), "INVALID_ARGUMENT"),
    (lambda p, pa: setattr(pa, "sort", 7), "INVALID_ARGUMENT"),
    (lambda p, pa: setattr(pa, "select", 1), "INVALID_ARGUMENT"),          # TOPP with top_p = 0
    (lambda p, pa: (setattr(pa, "select", 1), setattr(pa, "top_p", 1.01)), "INVALID_ARGUMENT"),
    (lambda p, pa: setattr(pa, "select", 2), "INVALID_ARGUMENT"),
    (lambda p, pa: setattr(pa, "comp", 3), "INVALID_ARGUMENT"),
])
def test_validation_errors(ba, mutate, code):
    q, k, v = _meta(1, 4, 2, 1000, 128)
    p, pa = ba.make_problem(q, k, v), ba.make_params()
    mutate(p, pa)
    with pytest.raises(ba.BaError, match=code):
        ba.selection_sizes(p, pa)


def test_select_rejects_bad_pointers_before_launch(ba):
    """Validation is synchronous: a NULL tensor pointer is reported without any
    CUDA call (works on a machine with no GPU)."""
    q, k, v = _meta(1, 2, 2, 256, 128)
    p, pa = ba.make_problem(q, k, v), ba.make_params()
    lib = ba.load()
    sel = ba.SelectionC()
    st = lib.ba_select(ctypes.byref(p), ctypes.byref(pa), None, None, None, ctypes.byref(sel), None, 0, None)
    assert lib.ba_status_string(st).decode() == "BA_ERR_INVALID_ARGUMENT"
    assert b"q is NULL" in lib.ba_last_error()
    # misaligned stride
    p.q_stride[2] = 130
    st = lib.ba_dense_attn(ctypes.byref(p), ctypes.byref(pa), ctypes.c_void_p(256), ctypes.c_void_p(256),
                           ctypes.c_void_p(256), ctypes.c_void_p(256), None, None)
    assert lib.ba_status_string(st).decode() == "BA_ERR_SHAPE_MISMATCH"


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2605_19726_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
                assert "ba_oracle" not in src, f


def test_no_cpu_fallback_without_library(tmp_path):
    """With the .so missing the binding raises instead of computing anything."""
    code = ("import paper_2605_19726_b200.baatt as b, os; b.LIB_PATH = '/nonexistent/libbaatt.so'; b._lib = None\n"
            "try:\n b.load()\nexcept b.BaError as e:\n print('RAISED', e)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert "RAISED" in r.stdout


def test_kernel_routing(ba):
    """bf16, d = 128, B in {64, 128} must run a tcgen05 kernel (never the SIMT path):
    the ping-pong pair kernel for B = 128, the dual-tile kernel for B = 64."""
    q, k, v = _meta(1, 32, 8, 131072, 128)
    assert ba.attention_kernel_name(q, k, v, 128) == "attn_sm100_tcgen05_pp"
    q, k, v = _meta(1, 32, 8, 1 << 21, 128)  # N_k > 8192: beyond the pair kernel's bitmask
    assert ba.attention_kernel_name(q, k, v, 128) == "attn_sm100_tcgen05"
    q, k, v = _meta(1, 28, 28, 65536, 128)
    assert ba.attention_kernel_name(q, k, v, 64) == "attn_sm100_tcgen05_dual64"
    q, k, v = _meta(1, 1, 1, 1024, 64, torch.float32)
    assert ba.attention_kernel_name(q, k, v, 64) == "attn_simt"


def test_exact_compensation_workspace(ba):
    """BA_COMP_EXACT (NEXT-4) carves the per-block covariances [b, H, N, d, d]
    fp64 of both sides from the select workspace."""
    lib = ba.load()
    q, k, v = _meta(1, 4, 2, 2048, 128)
    p = ba.make_problem(q, k, v)
    diag = lib.ba_select_workspace_size(ctypes.byref(p), ctypes.byref(ba.make_params(comp="diag")))
    exact = lib.ba_select_workspace_size(ctypes.byref(p), ctypes.byref(ba.make_params(comp="exact")))
    n = 2048 // 128
    assert exact - diag >= 8 * 128 * 128 * n * (4 + 2)


def test_units_validation_before_launch(ba):
    """ba_sparse_attn_units checks its unit range and output list synchronously
    (nothing is launched, so this runs without a GPU)."""
    q, k, v = _meta(1, 4, 2, 1000, 128)
    p, pa = ba.make_problem(q, k, v), ba.make_params()
    lib = ba.load()
    sel = ba.SelectionC()
    n_units = 4 * ((1000 + 127) // 128)
    outs = (ctypes.c_void_p * 1)(ctypes.c_void_p(256))
    for u0, u1 in ((-1, 3), (5, 4), (0, n_units + 1)):
        st = lib.ba_sparse_attn_units(ctypes.byref(p), ctypes.byref(pa), ctypes.byref(sel), u0, u1, outs, 1, None, None)
        assert lib.ba_status_string(st).decode() == "BA_ERR_INVALID_ARGUMENT"
        assert b"unit range" in lib.ba_last_error()
    st = lib.ba_sparse_attn_units(ctypes.byref(p), ctypes.byref(pa), ctypes.byref(sel), 0, n_units, outs, 9, None, None)
    assert b"n_out" in lib.ba_last_error()
    st = lib.ba_sparse_attn_units(ctypes.byref(p), ctypes.byref(pa), ctypes.byref(sel), 0, n_units, outs, 1, None, None)
    assert lib.ba_status_string(st).decode() == "BA_ERR_INVALID_ARGUMENT"  # empty selection struct


def test_no_silent_simt_for_bf16_d128(ba):
    """bf16 with head_dim 128 always runs a tcgen05 kernel; beyond their N_k <= 32768
    bitmask the attention calls return BA_ERR_UNSUPPORTED before any launch (no
    silent SIMT fallback), and ba_select refuses N_k above its shared-memory
    top-kappa capacity (28672) the same way.  Fake (never dereferenced) device
    pointers: validation happens before any CUDA call."""
    lib = ba.load()
    q, k, v = _meta(1, 1, 1, 32769 * 128, 128)
    assert ba.attention_kernel_name(q, k, v, 128) == ""
    p, pa = ba.make_problem(q, k, v), ba.make_params()
    fake = ctypes.c_void_p(1 << 20)
    st = lib.ba_dense_attn(ctypes.byref(p), ctypes.byref(pa), fake, fake, fake, fake, None, None)
    assert lib.ba_status_string(st).decode() == "BA_ERR_UNSUPPORTED"
    assert b"32768" in lib.ba_last_error()
    sel = ba.SelectionC()
    for f in ("perm_q", "perm_k", "q_sorted", "k_sorted", "v_sorted", "kv_index", "kv_count"):
        setattr(sel, f, 1 << 20)
    st = lib.ba_sparse_attn(ctypes.byref(p), ctypes.byref(pa), ctypes.byref(sel), fake, None, None)
    assert lib.ba_status_string(st).decode() == "BA_ERR_UNSUPPORTED"
    q, k, v = _meta(1, 1, 1, 28673 * 128, 128)
    p = ba.make_problem(q, k, v)
    st = lib.ba_select(ctypes.byref(p), ctypes.byref(pa), fake, fake, fake, ctypes.byref(sel), fake, 1 << 40, None)
    assert lib.ba_status_string(st).decode() == "BA_ERR_UNSUPPORTED"
    assert b"28672" in lib.ba_last_error()
    # bf16 head_dim 64 has no tcgen05 variant: the documented SIMT route, named as such
    q, k, v = _meta(1, 2, 2, 4096, 64)
    assert ba.attention_kernel_name(q, k, v, 128) == "attn_simt"
