"""Reference in the loop: INTEGRATION.md §2's solver swap executed against the
REAL reference package.

The unmodified reference (``mlmc_parareal``, pure Python) is installed into
``baseline/_ref`` by ``scripts/install_reference.sh`` (the offline
``pip install --target`` of /root/reference/pkg; git-ignored, it travels to the
GPU box with the snapshot).  Its own ``MachineFamily.evaluate``
(models.py:389-411) drives the reference's own Steinmetz circuit and synthetic
bar-machine builders (models.py:217-302, families :431-453) twice:

  * as shipped (CPU: dense LU, timeint.py:64-75);
  * with ``implicit_euler_solve`` / ``propagate`` / ``parareal_solve``
    replaced by this package's GPU mirrors — in ``mlmc_parareal.models`` too,
    which binds ``implicit_euler_solve`` at import (models.py:22), while
    ``parareal_solve`` is looked up lazily (models.py:400).

Per sample: Q within 1e-9 (Steinmetz: direct LU in another operation order,
step-matrix condition ~1e7) or 1e-8 (synthetic machine: Jacobi-PCG at the
stated tolerance), Parareal K equal.  Skipped when baseline/_ref is absent.
"""

import importlib
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "mlmc_parareal")):
        pytest.skip("reference not installed (scripts/install_reference.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    models = importlib.import_module("mlmc_parareal.models")
    timeint = importlib.import_module("mlmc_parareal.timeint")
    parareal = importlib.import_module("mlmc_parareal.parareal")
    assert os.path.dirname(models.__file__).startswith(REF)
    return models, timeint, parareal


def _swap(monkeypatch, ref):
    """INTEGRATION.md §2."""
    from paper_2507_19246_b200 import parareal as gpu_parareal
    from paper_2507_19246_b200 import timeint as gpu_timeint
    models, timeint, parareal = ref
    monkeypatch.setattr(timeint, "implicit_euler_solve", gpu_timeint.implicit_euler_solve)
    monkeypatch.setattr(timeint, "propagate", gpu_timeint.propagate)
    monkeypatch.setattr(models, "implicit_euler_solve", gpu_timeint.implicit_euler_solve)
    monkeypatch.setattr(parareal, "parareal_solve", gpu_parareal.parareal_solve)


CASES = {
    # family builder, hierarchy, horizon, Parareal (M, dt_coarse, tol, K_max), tolerance
    "steinmetz": ("steinmetz_family", [1e-3, 1e-4], 0.02, (10, 1e-3, 1e-8, 10), 1e-9),
    "synthetic": ("synthetic_family", [1e-3, 2.5e-4], 0.02, (4, 1e-3, 1e-8, 4), 1e-8),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_reference_family_evaluate_with_gpu_solvers(cuda, ref, name, monkeypatch):
    from paper_2507_19246_b200.mlmc import RandomStream
    models, timeint, parareal = ref
    builder, dts, horizon, (m, dtc, tol, kmax), rtol = CASES[name]
    kw = {"n_dof": 64} if name == "synthetic" else {}
    fam = getattr(models, builder)(models.make_hierarchy(dts), horizon=horizon, **kw)
    pcfg = parareal.PararealConfig(m, dts[-1], dtc, tol, kmax)
    params = [models.draw_parameters(fam.uncertain, RandomStream(0, lvl, k))
              for lvl in range(len(dts)) for k in (1, 2)]
    levels = [lvl for lvl in range(len(dts)) for _ in (1, 2)]
    top = len(dts) - 1

    def run_all():
        out = []
        for p, lvl in zip(params, levels):
            rec = fam.evaluate(p, fam.hierarchy[lvl], pcfg if lvl == top else None)
            out.append((rec.q, rec.parareal_iterations))
        return out

    cpu = run_all()                      # the reference as shipped
    _swap(monkeypatch, ref)
    assert models.implicit_euler_solve.__module__.startswith("paper_2507_19246_b200")
    gpu = run_all()                      # the same calls through the GPU mirrors
    for (qc, kc), (qg, kg), lvl in zip(cpu, gpu, levels):
        assert kc == kg, (name, lvl, kc, kg)
        assert abs(qg - qc) <= rtol * abs(qc), (name, lvl, qg, qc)
