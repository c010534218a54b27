"""bench.py's reference arm (the CPU oracle timed on the host cores) keeps the
driver's JSON contract; runs on CPU (no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "A", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def _bench(args, env=None, timeout=600):
    r = subprocess.run([sys.executable, "bench.py"] + args, capture_output=True, text=True, cwd=ROOT,
                       timeout=timeout, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_product_line_config_T():
    """The product arm's JSON line on the small config (fp32 SIMT path): every
    contract key, per-stage percentiles, a positive device-timed value and a
    launch count from the library."""
    d = _bench(["--config", "T", "--steps", "3", "--warmup", "3", "--no-cpu"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "stage_ms"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["stage_ms"]) == {"ba_select", "ba_sparse_attn"}


@pytest.mark.gpu
def test_bench_unit_split_single_rank():
    """--shard units on one rank (the uneven-split path of SURVEY 8(e): units
    covering every head, ba_sparse_attn_units) produces the same work as the
    default run."""
    base = _bench(["--config", "T", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-dense"])
    d = _bench(["--config", "T", "--shard", "units", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e",
                "--no-dense"])
    assert d["scaling"] == "strong" and d["config"]["parallelism"].startswith("unit-parallel x1")
    assert d["flops_per_step_per_rank"] == base["flops_per_step_per_rank"]


@pytest.mark.parametrize("args,par", [
    (["--config", "C", "--seq-len", "2048", "--gpus", "2"], "head-parallel x2"),
    (["--config", "C", "--seq-len", "1500", "--gpus", "4"], "head-parallel x4"),
    (["--config", "M", "--seq-len", "1024", "--gpus", "3"], "unit-parallel x3"),
])
def test_bench_gpus_n_self_launches_ranks(args, par):
    """`bench.py --gpus N` outside torchrun re-launches itself as N ranks
    (torch.distributed.run) and defaults to the head-parallel strong-scaling split
    with the output collective in the step; --dry-run runs the same launcher,
    partition and reassembly on CPU (gloo) ranks with a stand-in kernel and
    checks that every rank ends up with the whole layer's O."""
    d = _bench(args + ["--dry-run", "--steps", "2", "--warmup", "1"], timeout=300)
    n = int(args[args.index("--gpus") + 1])
    assert d["n_gpus"] == n and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith(par)
    assert d["dry_run"] == "reassembled O equals the 1-rank layout on every rank"
    assert d["value"] is None  # a dry run is never a measurement
