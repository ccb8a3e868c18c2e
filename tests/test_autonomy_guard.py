"""Compile-time autonomy guard of the model layer (-m "not gpu"; nvcc
cross-compiles for sm_100a without a GPU).

The fixed-step Tsit5 loop passes t = 0 to its stages, EM/SIEA evaluate the
drift at t = 0, the Verner stages use the step's start time and the
Rosenbrock/Rodas steps drop the β_i·h²·∂f/∂t term of the general form
(P:125-136). Each of those paths static_asserts that the model declares
`autonomous = true`, so a time-dependent model cannot silently compile into
them."""
import shutil
import subprocess
from pathlib import Path

import pytest

CSRC = Path(__file__).resolve().parents[1] / "paper_2304_06835_b200" / "csrc"

PROBE = r'''
#include "tsit5.cuh"
#include "ros23.cuh"
#include "rodas.cuh"
#include "verner.cuh"
#include "em.cuh"
namespace ens {
struct TimeDep {            // u' = t·u (∂f/∂t ≠ 0)
  static constexpr int n = 1, m = 1, nw = 1;
  AUTONOMOUS_DECL
  template <class T> __device__ static void f(const T (&y)[1], const T (&)[1], T t, T (&o)[1]) { o[0] = t * y[0]; }
  template <class T> __device__ static void jac(const T (&)[1], const T (&)[1], T t, T (&J)[1][1]) { J[0][0] = t; }
  template <class T> __device__ static void g(const T (&y)[1], const T (&)[1], T, T (&b)[1]) { b[0] = y[0]; }
};
}  // namespace ens
__global__ void probe(double* x) {
  double par[1] = {1.0}, u[1] = {x[0]}, F0[1] = {x[1]}, un[1], F2[1], k1[1], k2[1], E[1];
  PROBE_BODY
  x[2] = un[0];
}
'''

BODIES = {
    "rosenbrock23": "ens::ros23_step<ens::TimeDep, double>(par, 0.0, 0.1, u, F0, un, F2, k1, k2, E);",
    "rodas5": "double K[8][1]; (void)F2; (void)k1; (void)k2; (void)E;"
              " ens::rodas_step<ens::Rodas5Tab, ens::TimeDep, double>(par, 0.0, 0.1, u, F0, un, K);",
    "vern7": "double K[10][1]; K[0][0] = F0[0]; (void)F2; (void)k1; (void)k2;"
             " ens::verner_step<ens::Vern7Tab, ens::TimeDep, double, true>(par, 0.0, 0.1, u, K, un, E);",
    "tsit5_fixed": "(void)F2; (void)k1; (void)k2; (void)E; un[0] = u[0];"
                   " auto kern = ens::tsit5_fixed_kernel<ens::TimeDep, double, 0>; (void)kern;",
    "em": "(void)F2; (void)k1; (void)k2; (void)E; un[0] = u[0];"
          " auto kern = ens::em_kernel<ens::TimeDep, double, false>; (void)kern;",
}


def _nvcc():
    for c in ["/usr/local/cuda/bin/nvcc", shutil.which("nvcc")]:
        if c and Path(c).exists():
            return c
    pytest.skip("nvcc not available")


def _compile(tmp_path, body, decl):
    src = tmp_path / "probe.cu"
    src.write_text(PROBE.replace("AUTONOMOUS_DECL", decl).replace("PROBE_BODY", body))
    r = subprocess.run([_nvcc(), "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I", str(CSRC),
                        "-I", str(CSRC.parents[1] / "include"), "-c", "-o", str(tmp_path / "probe.o"), str(src)],
                       capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.parametrize("path", sorted(BODIES))
def test_time_dependent_model_does_not_compile(tmp_path, path):
    rc, log = _compile(tmp_path, BODIES[path], "")
    assert rc != 0 and "elides the time dependence" in log, log[-2000:]
    rc, log = _compile(tmp_path, BODIES[path], "static constexpr bool autonomous = false;")
    assert rc != 0 and "elides the time dependence" in log, log[-2000:]


def test_declared_autonomous_model_compiles(tmp_path):
    """Control: the same probe compiles once the model declares autonomy."""
    rc, log = _compile(tmp_path, BODIES["rosenbrock23"], "static constexpr bool autonomous = true;")
    assert rc == 0, log[-2000:]
