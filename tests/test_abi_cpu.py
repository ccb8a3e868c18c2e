"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports every
symbol include/ens.h declares, and rejects invalid arguments synchronously with
the documented status codes before touching the device."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2304_06835_b200 as ens

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    src = (ROOT / "include" / "ens.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s+(ens_[a-z_0-9]+|ensemble_[a-z_0-9]+)\s*\(",
                                 src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert "ensemble_solve" in names and "ens_generate_inputs" in names and len(names) >= 10
    L = ens.lib()
    for nm in names:
        assert hasattr(L, nm), nm
    assert set(names) == set(ens.EXPORTS)
    assert b"sm_100a" in L.ens_version()


def test_model_dims_and_status_strings():
    assert ens.model_dims("lorenz") == (3, 3, 0)
    assert ens.model_dims("robertson") == (3, 3, 0)
    assert ens.model_dims("lorenz_sde_add") == (3, 4, 3)
    assert ens.model_dims("gbm") == (3, 2, 3)
    assert ens.model_dims("harmonic") == (2, 1, 0)
    for s in range(10):
        assert len(ens.status_string(s)) >= 2 and ens.status_string(s) != "unknown status"
    n = ctypes.c_int32()
    assert ens.lib().ens_model_dims(99, ctypes.byref(n), None, None) == 1


def test_workspace_bytes_host_only():
    a = ens.workspace_bytes("lorenz", "tsit5", __import__("torch").float32, 1000)
    b = ens.workspace_bytes("lorenz", "tsit5", __import__("torch").float32, 1000, n_saveat=100, stats=True)
    c = ens.workspace_bytes("gbm", "em", __import__("torch").float64, 10**6, n_saveat=11, stats=True)
    assert 256 <= a < b and c >= 11 * 3 * (10**6 // 256) * 24


def _call(model, alg, dtype=0, N=16, t0=0.0, tf=1.0, dt=1e-3, **o):
    L = ens.lib()
    opt = ens._Options()
    keep = []
    for k, v in o.items():
        if k == "saveat":
            arr = np.ascontiguousarray(v, dtype=np.float64)
            keep.append(arr)
            opt.saveat = arr.ctypes.data
            opt.n_saveat = arr.size
        else:
            setattr(opt, k, v)
    out = ens._Output()
    fake = ctypes.c_void_p(0x1000)   # never dereferenced: validation returns first
    out.u_out = fake; out.workspace = None; out.workspace_bytes = 0
    return L.ensemble_solve(ens.MODELS[model], ens.ALGS[alg], dtype, N, fake, fake, t0, tf, dt, ctypes.byref(opt),
                            ctypes.byref(out), None)


@pytest.mark.parametrize("kw,status", [
    (dict(model="lorenz", alg="tsit5", N=0), 1),                                   # N < 1
    (dict(model="lorenz", alg="em"), 2),                                           # EM on an ODE
    (dict(model="gbm", alg="tsit5"), 2),                                           # ODE alg on an SDE
    (dict(model="gbm", alg="em", adaptive=1, abstol=1e-6), 3),                     # P:335 fixed-step SDEs only
    (dict(model="lorenz", alg="tsit5", adaptive=1, abstol=0.0), 4),
    (dict(model="lorenz", alg="tsit5", adaptive=1, abstol=1e-6, reltol=-1.0), 4),
    (dict(model="lorenz", alg="tsit5", t0=1.0, tf=1.0), 5),
    (dict(model="lorenz", alg="tsit5", dt=0.0), 5),
    (dict(model="lorenz", alg="tsit5", dt=float("nan")), 5),
    (dict(model="lorenz", alg="tsit5", saveat=[0.2, 0.1]), 6),                    # unsorted
    (dict(model="lorenz", alg="tsit5", saveat=[0.5, 1.5]), 6),                    # outside [t0, tf]
    (dict(model="gbm", alg="em", saveat=[0.00015]), 6),                           # off the EM grid
    (dict(model="lorenz", alg="tsit5"), 7),                                        # no workspace
    (dict(model="gbm", alg="rodas4"), 2),                                          # Rodas4 on an SDE
    (dict(model="ball", alg="rodas4", adaptive=1, abstol=1e-6), 8),                # events: Tsit5 only (R18)
    (dict(model="pollu", alg="rodas4", dtype=0), 8),                               # POLLU: fp64 only
    (dict(model="lorenz", alg="rodas4", adaptive=1, abstol=-1.0), 4),
    (dict(model="lorenz", alg="rodas4"), 7),                                       # valid up to the workspace
    (dict(model="lorenz", alg="vern7", saveat=[0.00015]), 7),                      # fixed Vern7: any τ (R24)
    (dict(model="lorenz", alg="vern7", adaptive=1, abstol=1e-8, saveat=[0.00015]), 7),   # adaptive: any τ
    (dict(model="gbm", alg="vern7"), 2),
    (dict(model="lorenz", alg="rodas5", saveat=[0.00015]), 7),                     # fixed Rodas5: any τ (R24)
    (dict(model="ball", alg="rodas5", adaptive=1, abstol=1e-6), 8),
    (dict(model="lorenz", alg="vern9", saveat=[0.00015]), 7),
    (dict(model="lorenz", alg="em", saveat=[0.00015]), 2),                          # EM: lorenz is an ODE model
    (dict(model="pollu", alg="vern9", dtype=1), 8),                                # n = 20: stiff solvers only
    (dict(model="lorenz", alg="tsit5", N=16, out_ld=8), 1),                        # out_ld < N
    (dict(model="lorenz", alg="tsit5", N=16, out_ld=32), 7),                       # wider rows: valid
])
def test_validation_statuses(kw, status):
    assert _call(**kw) == status


def test_generate_inputs_validation():
    L = ens.lib()
    fake = ctypes.c_void_p(0x1000)
    assert L.ens_generate_inputs(ens.MODELS["robertson"], 0, 1, 0, 10, 10, None, fake, fake, None) == 8
    assert L.ens_generate_inputs(ens.MODELS["lorenz"], 0, 7, 0, 10, 10, None, fake, fake, None) == 1
    assert L.ens_generate_inputs(ens.MODELS["lorenz"], 0, 0, 0, 0, 10, None, fake, fake, None) == 1


def test_ctypes_structs_match_the_header(tmp_path):
    """The binding's ctypes mirrors of ens_options / ens_output have the C header's
    size and field offsets (compiled from include/ens.h with the host compiler)."""
    import ctypes
    import shutil
    import subprocess

    import paper_2304_06835_b200 as ens
    cxx = shutil.which("g++") or shutil.which("c++")
    if not cxx:
        import pytest
        pytest.skip("no host C++ compiler")
    inc = ROOT / "include"
    fields = [f for f, _ in ens._Options._fields_]
    ofields = [f for f, _ in ens._Output._fields_]
    src = tmp_path / "layout.cpp"
    src.write_text('#include <cstdio>\n#include <cstddef>\n#include "ens.h"\nint main(){\n'
                   + 'printf("%zu\\n", sizeof(ens_options));\n'
                   + "".join(f'printf("%zu\\n", offsetof(ens_options, {f}));\n' for f in fields)
                   + 'printf("%zu\\n", sizeof(ens_output));\n'
                   + "".join(f'printf("%zu\\n", offsetof(ens_output, {f}));\n' for f in ofields)
                   + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.check_call([cxx, "-I", str(inc), "-o", str(exe), str(src)])
    vals = [int(x) for x in subprocess.check_output([str(exe)], text=True).split()]
    want = ([ctypes.sizeof(ens._Options)] + [getattr(ens._Options, f).offset for f in fields]
            + [ctypes.sizeof(ens._Output)] + [getattr(ens._Output, f).offset for f in ofields])
    assert vals == want, (vals, want)
