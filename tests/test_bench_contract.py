"""bench.py's reference arm (the driver's `--impl reference` line) runs on the
CPU: it must print exactly one JSON line with the contract's keys, timed on
the reference's own CPU path (oracle/_ref when built, else the C port)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--workload", "cfg0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["metric"].startswith("cell-updates/s")


def test_reference_arm_nonzero_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--gpus", "2"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == ""


def _torchrun_bench(n, port, *extra):
    env = dict(os.environ, HYDRO_BENCH_SHARED_GPU="1")
    return subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                           f"--master-port={port}", os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                           "--steps", "1", "--warmup", "1", "--no-variants", *extra],
                          capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)


import pytest  # noqa: E402


@pytest.mark.gpu
def test_multi_rank_bench_code_path(gpu):
    """The driver's N>1 launch (torchrun, one process per GPU): every rank runs
    the slab driver with the peer-memory halo and rank 0 alone prints one
    contract line.  Run here with all ranks sharing cuda:0 and gloo for the
    host-side dt allreduce (HYDRO_BENCH_SHARED_GPU), so it checks the code
    path, not the speed; 3 ranks give the middle slab two neighbours."""
    out = _torchrun_bench(3, 29641)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    # BASELINE config 3 strong-scaled over 3 row slabs: the same global grid,
    # so the bitwise state's digest -- chained over the ranks' slabs -- is the
    # reference's, and the tolerance headline is within 1e-12 of it
    assert d["n_gpus"] == 3 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["cells"] == 16384 * 16384
    assert d["bitwise_digest"] == "b14afe9de695c517"
    assert 0 < d["max_rel_vs_bitwise"] <= 1e-12
    assert "peer-memory" in d["config"]["halo"]
    for key in ("roofline", "e2e", "gpu_launches", "clocks", "ms_per_step"):
        assert key in d, key


@pytest.mark.gpu
def test_single_gpu_bench_line_carries_the_contract_keys(gpu):
    """The driver's default N=1 run (config 3, tolerance headline): one JSON
    line with the base contract's keys plus roofline, e2e (host buffers),
    clocks, gpu_launches, the bitwise state's digest (the reference's
    b14afe9de695c517) and the headline's measured max_rel against it."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1",
                          "--warmup", "1", "--no-variants", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["dtype"] == "f64" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1
    assert d["config"]["math"] == "tolerance" and d["config"]["cells"] == 16384 * 16384
    assert d["bitwise_digest"] == "b14afe9de695c517"
    assert 0 < d["max_rel_vs_bitwise"] <= 1e-12
    assert d["gpu_launches"] > 0


@pytest.mark.gpu
def test_bench_variants_tolerance_within_bound(gpu):
    """The variants of a bitwise-headline run on config 1: the headline keeps
    the reference's digest, exact-10 the oracle's (tests/golden/
    golden_full.json), and both tolerance lines are within 1e-12 of their
    bitwise states."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1",
                          "--warmup", "1", "--no-cpu-baseline", "--workload", "cfg1",
                          "--math", "bitwise"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.strip().startswith("{")][0])
    assert d["config"]["math"] == "bitwise"
    assert d["result_digest"] == d["golden_digest"] == "e00cb4cfa888c325"
    assert d["flux_variants"]["exact10_bitwise"]["result_digest"] == "5bba80ba4684d325"
    for v in (d["math_variants"]["tolerance"], d["flux_variants"]["exact10_tolerance"]):
        assert v["value"] > 0
        assert 0 < v["max_rel_vs_bitwise"] <= 1e-12, v["max_rel_vs_bitwise"]
    for wl in ("cfg2",):
        sec = d["secondary"][wl]
        assert sec["bitwise"]["result_digest"] == sec["bitwise"]["golden_digest"]
        assert 0 < sec["tolerance"]["max_rel_vs_bitwise"] <= 1e-12
