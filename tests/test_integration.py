"""The drop-in: the reference's own command surface (RunConfig, make_case,
grid_checksum/format_checksum, error convention) with a "gpu" strategy that
goes through include/hydro/gpu_strategy.hpp and the C-ABI
(integration/hydrobench_gpu.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "hydrobench_gpu")
README_LINE = ("checksum b4593af8ee8e4e25  rho=2304 mom_x=0 mom_y=-3.4208746946262636e-15 "
               "ener=2304.0230000000001")  # proj/README.md:98-101

needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="integration driver not built")


def run(*args):
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)


@needs_bin
def test_reference_strategy_reproduces_readme_line():
    out = run("run", "--case", "blast", "--nx", "48", "--ny", "48", "--steps", "5",
              "--strategy", "task_graph", "--workers", "4")
    assert out.returncode == 0, out.stderr
    assert out.stdout.splitlines()[1] == README_LINE


@needs_bin
def test_error_convention_for_bad_flags():
    out = run("run", "--case", "nope", "--strategy", "gpu")
    assert out.returncode == 1
    assert out.stderr.startswith("error: config: unknown case")


@needs_bin
@pytest.mark.gpu
def test_gpu_strategy_reproduces_readme_line():
    out = run("run", "--case", "blast", "--nx", "48", "--ny", "48", "--steps", "5",
              "--strategy", "gpu")
    assert out.returncode == 0, out.stderr
    assert out.stdout.splitlines()[0].startswith("case=blast 48x48 steps=5 strategy=gpu")
    assert out.stdout.splitlines()[1] == README_LINE


@needs_bin
@pytest.mark.gpu
@pytest.mark.parametrize("case,n,steps,strategy", [("blast", 64, 10, "coarse_grain"),
                                                   ("sod", 128, 40, "sequential")])
def test_gpu_strategy_equals_cpu_strategy(case, n, steps, strategy):
    args = ["--case", case, "--nx", str(n), "--ny", str(n), "--steps", str(steps)]
    cpu = run("run", *args, "--strategy", strategy, "--workers", "4" if strategy != "sequential" else "1")
    gpu = run("run", *args, "--strategy", "gpu")
    assert cpu.returncode == 0 and gpu.returncode == 0, (cpu.stderr, gpu.stderr)
    assert cpu.stdout.splitlines()[1] == gpu.stdout.splitlines()[1]


@needs_bin
@pytest.mark.gpu
@pytest.mark.parametrize("gpus", [2, 3])
def test_gpu_strategy_row_slabs_equal_cpu_strategy(gpus):
    """--gpus N: the C++ adaptor's hydro_gpu_group path (all slabs on GPU 0
    here via --device 0) reproduces the reference's checksum line."""
    args = ["--case", "blast", "--nx", "96", "--ny", "80", "--steps", "12"]
    cpu = run("run", *args, "--strategy", "coarse_grain", "--workers", "4")
    gpu = run("run", *args, "--strategy", "gpu", "--gpus", str(gpus), "--device", "0")
    assert cpu.returncode == 0 and gpu.returncode == 0, (cpu.stderr, gpu.stderr)
    assert cpu.stdout.splitlines()[1] == gpu.stdout.splitlines()[1]


@needs_bin
@pytest.mark.gpu
def test_gpu_positivity_error_line_matches_reference():
    args = ["--case", "blast", "--nx", "64", "--ny", "64", "--steps", "5", "--cfl", "25"]
    cpu = run("run", *args, "--strategy", "sequential")
    gpu = run("run", *args, "--strategy", "gpu")
    assert cpu.returncode == gpu.returncode == 1
    assert cpu.stderr == gpu.stderr
    assert cpu.stderr.startswith("error: positivity: step ")


@needs_bin
def test_cpu_strategies_reject_the_gpu_only_flux():
    out = run("run", "--case", "blast", "--nx", "32", "--ny", "32", "--steps", "1",
              "--strategy", "sequential", "--flux", "exact10")
    assert out.returncode == 1
    assert out.stderr.startswith("error: config: the CPU strategies only have the HLLC flux")


@needs_bin
@pytest.mark.gpu
def test_gpu_strategy_exact10_flux_equals_oracle():
    """--flux exact10 through the C++ adaptor (GpuOptions::flux): the checksum
    digest equals the oracle's exact-10 run of the same case."""
    import numpy as np

    from oracle import oracle as O
    out = run("run", "--case", "sod_x", "--nx", "64", "--ny", "40", "--steps", "12",
              "--bc", "transmit", "--strategy", "gpu", "--flux", "exact10")
    assert out.returncode == 0, out.stderr
    digest = out.stdout.splitlines()[1].split()[1]
    ref = O.make_case("sod_x", 64, 40)
    with O.flux_mode("exact10"):
        O.run_sequential(ref, 12, "transmit")
    assert digest == f"{O.digest(ref):016x}"
    assert np.isfinite(ref.u).all()


@needs_bin
def test_cpu_strategies_reject_the_tolerance_math():
    out = run("run", "--case", "blast", "--nx", "32", "--ny", "32", "--steps", "1",
              "--strategy", "sequential", "--math", "tolerance")
    assert out.returncode == 1
    assert out.stderr.startswith("error: config: the CPU strategies only have the reference's arithmetic")


@needs_bin
@pytest.mark.gpu
@pytest.mark.parametrize("gpus", [1, 2])
def test_gpu_strategy_tolerance_math_totals(gpus):
    """--math tolerance through the C++ adaptor (GpuOptions::math, one context
    or a 2-slab group on GPU 0): the checksum line's conserved totals are the
    reference's within 1e-12 (relative, floored at 1)."""
    args = ["run", "--case", "blast", "--nx", "48", "--ny", "48", "--steps", "5"]
    ref = run(*args, "--strategy", "sequential")
    tol = run(*args, "--strategy", "gpu", "--math", "tolerance", "--gpus", str(gpus), "--device", "0")
    assert ref.returncode == 0 and tol.returncode == 0, tol.stderr

    def totals(out):
        fields = out.stdout.splitlines()[1].split()[2:]
        return [float(f.split("=")[1]) for f in fields]

    for a, b in zip(totals(ref), totals(tol)):
        assert abs(a - b) <= 1e-12 * max(abs(a), abs(b), 1.0)
