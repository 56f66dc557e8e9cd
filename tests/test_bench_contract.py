"""bench.py's driver contract on CPU: the reference arm (the oracle, timed on the host cores)
prints one JSON line with the keys the driver reads, on rank 0 only; under torchrun
(world 2) the other rank exits 0 without work or output.  The GPU arm is covered by the
round-end bench itself (it needs a B200)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _lines(out):
    return [json.loads(s) for s in out.splitlines() if s.startswith("{")]


def test_reference_arm_single_rank():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg2", "--steps", "2",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    (d,) = _lines(r.stdout)
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # cfg2: Q2 on 16^3 cells, (2*16+1)^3 DoFs
    assert d["config"]["n_dofs"] == 33 ** 3 and d["config"]["parallelism"] == "zslab1"


def test_reference_arm_world2_rank0_only():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--config", "cfg2", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout  # rank 1 prints nothing
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    # weak scaling: the z extent (and the DoF count) grows with the world size
    assert d["config"]["n_cells"] == [16, 16, 32] and d["config"]["n_dofs"] == 33 * 33 * 65
    assert d["config"]["parallelism"] == "zslab2"


@pytest.mark.parametrize("bad", [["--config", "nope"], ["--impl", "nope"]])
def test_bench_rejects_unknown_arguments(bad):
    r = subprocess.run([sys.executable, "bench.py", *bad], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0


def test_reference_arm_world2_default_is_strong_scaling_cfg5():
    # N > 1 without --config: BASELINE configs[4], the 256^3 Q4 cube split over the ranks
    env = dict(os.environ, OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29534", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    (d,) = _lines(r.stdout)
    assert d["scaling"] == "strong" and d["config"]["config"] == "cfg5q4"
    assert d["config"]["n_cells"] == [256, 256, 256] and d["config"]["n_dofs"] == 1025 ** 3


@pytest.mark.gpu
def test_main_arm_json_line_contract():
    # the driver's bench contract on a small config: one JSON line with the keys it reads, the
    # roofline / cpu_baseline / e2e / clocks objects, and a positive count of our own launches
    env = dict(os.environ, OMP_NUM_THREADS="4")
    r = subprocess.run([sys.executable, "bench.py", "--config", "cfg2", "--steps", "3", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and d["value"] > 0 and d["gpu_launches"] > 0
    ro = d["roofline"]
    assert ro["bound"] in ("hbm", "tensor", "alu") and 0 < ro["frac"] < 1 and ro["unit"] == "GB/s"
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_max_mhz"] and "reasons" in d["clocks"]
    assert d["identity_rows_exact"] is True
