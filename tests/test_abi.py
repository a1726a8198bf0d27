"""The C-ABI library loads and exports everything include/hydro_gpu.h declares,
and its host-only entry points agree with the oracle.  No device work here."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import paper_2106_13465_b200 as P
from oracle import oracle as O
from paper_2106_13465_b200 import _lib


def test_library_exports_every_declared_symbol():
    names = _lib.declared_symbols()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n)


def test_abi_version_and_status_strings():
    L = _lib.lib()
    assert L.hydro_gpu_abi_version() == 1
    want = ["ok", "config", "positivity", "protocol", "task-graph", "equivalence", "io",
            "validation", "cuda"]
    assert [L.hydro_gpu_status_string(k).decode() for k in range(9)] == want


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("bad", [dict(nx=3, ny=8), dict(nx=8, ny=3), dict(dx=0.0),
                                 dict(gamma=1.0), dict(bc=7), dict(flux=3),
                                 dict(row0=5, global_nx=8)])
def test_create_rejects_bad_config_without_device(bad):
    base = dict(nx=8, ny=8, dx=0.1, dy=0.1, gamma=1.4, cfl=0.8, bc=0, flux=0, device=-1,
                row0=0, global_nx=8, wall_lo=1, wall_hi=1)
    base.update(bad)
    cfg = _lib.Cfg(**base)
    ctx = C.c_void_p()
    assert _lib.lib().hydro_gpu_create(C.byref(cfg), C.byref(ctx)) == 1
    assert not ctx.value


@pytest.mark.parametrize("case,nx,ny,seed", [("blast", 48, 48, 0), ("blast", 37, 53, 0),
                                             ("corner_blast", 64, 32, 0), ("sod_x", 33, 17, 0),
                                             ("random", 40, 24, 2106), ("uniform", 9, 5, 0),
                                             ("sod", 4, 64, 0)])
def test_host_initialisers_and_digest_match_oracle(case, nx, ny, seed):
    g = P.make_case(case, nx, ny, seed=seed)
    o = O.make_case(case, nx, ny, seed=seed)
    assert (g.dx, g.dy) == (o.dx, o.dy)
    assert np.array_equal(g.planes, o.u)
    O.run_sequential(o, 3, "reflect")
    g2 = P.Grid2D(o.nx, o.ny, o.dx, o.dy, o.u.copy())
    assert P.grid_digest(g2) == O.digest(o)


def test_digest_sensitive_to_one_bit():
    # test_bench.cpp:154-174: checksum sensitivity
    g = P.make_case("random", 16, 16, seed=1)
    d0 = P.grid_digest(g)
    g.planes[3, 9, 9] = np.nextafter(g.planes[3, 9, 9], 10.0)
    assert P.grid_digest(g) != d0
    g.planes[3, 9, 9] = np.nextafter(g.planes[3, 9, 9], 0.0)
    assert P.grid_digest(g) == d0
    g.planes[0, 0, 5] = 123.0  # ghosts are not part of the digest
    assert P.grid_digest(g) == d0


def test_grid_mirror_rejects_bad_shapes():
    with pytest.raises(P.ConfigError):
        P.Grid2D(3, 8, 0.1, 0.1)
    with pytest.raises(P.ConfigError):
        P.make_case("nope", 8, 8)
    with pytest.raises(P.ConfigError):
        P.make_case("sod", 4, 6)


def test_error_cli_line_format():
    e = P.PositivityError(2, "step 0: column sweep strip 3: rho non-positive at strip cell 1")
    assert e.cli_line() == ("error: positivity: step 0: column sweep strip 3: rho non-positive "
                            "at strip cell 1")
