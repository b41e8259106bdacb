"""Small workloads that exercise every libmlmcp kernel family once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  fused     SM-resident device-scheduled estimate launch (fused_kernel: the
            lock-free device FIFO of Parareal chain steps), steady-state COCG,
            assembly, draws, K7
  small     separate SM-resident launches (small_propagate / coarse / defect /
            finalize / energy)
  cluster   thread-block-cluster kernel with DSMEM halo exchange + cluster
            coarse sweep (MLMCP_STREAM_IMPL=3)
  tile      HBM-streaming tile kernels chained by programmatic dependent
            launch (MLMCP_STREAM_IMPL=4), ragged grid
  coop      cooperative grid-resident kernel (MLMCP_STREAM_IMPL=2)
  ell       two-launch ELL kernels (MLMCP_STREAM_IMPL=1)
  graph     device-driven step loop (conditional graph nodes)
  direct    Steinmetz 3x3 direct-LU path with Parareal

Usage:  python scripts/sanitize_cases.py <case>   (each case ends with "ok")
Results are checked against the CPU oracle so a silent corruption fails too.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _quad4_family(n, dts, path="auto"):
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.configs import T
    from paper_2507_19246_b200.models import (EddyCurrentFamily, ParameterVector, QoIKind,
                                              UncertainInput, make_hierarchy)
    nominal = np.array([fe.NU0] * 4 + [fe.SIGMA0] * 4)
    return EddyCurrentFamily("quad4", UncertainInput(ParameterVector("quad4", nominal), 0.1),
                             make_hierarchy([d * T for d in dts]), T, n, "quad4",
                             QoIKind.MAGNETIC_ENERGY_T, device="cuda:0", path=path)


def _blocks8_family(n, dts, path="stream"):
    from paper_2507_19246_b200 import fe
    from paper_2507_19246_b200.configs import T
    from paper_2507_19246_b200.models import (EddyCurrentFamily, ParameterVector, QoIKind,
                                              UncertainInput, make_hierarchy)
    nominal = np.array([fe.NU0] * 8 + [fe.SIGMA0] * 8)
    return EddyCurrentFamily("blocks8", UncertainInput(ParameterVector("blocks8", nominal), 0.1),
                             make_hierarchy([d * T for d in dts]), T, n, "blocks8",
                             QoIKind.MAGNETIC_ENERGY_T, device="cuda:0", path=path)


def _check(fam, n, layout, lvl, params, q, pr=None):
    from oracle import mlmc_oracle as mo
    from paper_2507_19246_b200.configs import T
    dts = tuple(s.dt for s in fam.hierarchy)
    cfg = mo.OracleConfig("san", n, layout, T, dts, (1,) * len(dts), "energy_T", parareal=pr)
    prob = mo.FEProblem(n, layout)
    for i, p in enumerate(params):
        ref = mo.coupled(prob, cfg, lvl, p)[0]
        assert abs(q[i] - ref) <= 1e-8 * abs(ref), (i, q[i], ref)


def case_fused():
    from paper_2507_19246_b200.configs import T
    from paper_2507_19246_b200.mlmc import FixedSamples, draw_level, mlmc_estimate
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = _quad4_family(8, (1 / 32, 1 / 64, 1 / 128))
    pc = PararealConfig(4, T / 128, T / 16, 1e-8, 4)
    mlmc_estimate(fam, policy=FixedSamples((5, 3, 3)), parareal_cfg=pc, seed=0)
    d = [draw_level(fam.uncertain, 0, lvl, range(1, 4)) for lvl in range(3)]
    out = fam.run_levels(d, pc)
    fam.check_status()
    _check(fam, 8, "quad4", 2, d[2], out[2].q_l.cpu().numpy(), pr=(4, T / 16, 1e-8, 4))


def case_small():
    from paper_2507_19246_b200.configs import T
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = _quad4_family(16, (1 / 32, 1 / 64))
    d = [draw_level(fam.uncertain, 0, lvl, range(1, 4)) for lvl in range(2)]
    out = fam.run_levels(d, PararealConfig(4, T / 64, T / 16, 1e-8, 3), fused=False)
    fam.check_status()
    _check(fam, 16, "quad4", 0, d[0], out[0].q_l.cpu().numpy())


def _stream_case(impl, n=72, extra=None):
    os.environ["MLMCP_STREAM_IMPL"] = impl
    for k, v in (extra or {}).items():
        os.environ[k] = v
    from paper_2507_19246_b200.configs import T
    from paper_2507_19246_b200.mlmc import draw_level
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = _blocks8_family(n, (1 / 16, 1 / 32))
    d = draw_level(fam.uncertain, 0, 0, range(1, 3))
    out = fam.run_levels([d], levels=[0])[0]
    fam.check_status()
    _check(fam, n, "blocks8", 0, d, out.q_l.cpu().numpy())
    pp = draw_level(fam.uncertain, 0, 1, range(1, 2))
    b = fam.run_levels([pp], PararealConfig(4, T / 32, T / 4, 1e-8, 2), levels=[1])[0]
    fam.check_status()
    _check(fam, n, "blocks8", 1, pp, b.q_l.cpu().numpy(), pr=(4, T / 4, 1e-8, 2))


def case_cluster():
    _stream_case("3", n=64)


def case_tile():
    _stream_case("4", n=72)


def case_coop():
    _stream_case("2", n=40)


def case_ell():
    _stream_case("1", n=40)


def case_graph():
    _stream_case("4", n=72, extra={"MLMCP_STREAM_GRAPH": "1"})


def case_direct():
    from paper_2507_19246_b200 import machines as mc
    from paper_2507_19246_b200.models import make_hierarchy
    from paper_2507_19246_b200.parareal import PararealConfig
    fam = mc.steinmetz_family(make_hierarchy([1e-3, 1e-4]), horizon=0.01, device="cuda:0")
    p = np.array([fam.uncertain.nominal.values] * 2)
    fam.evaluate_batch(p, fam.hierarchy[0])
    fam.evaluate_batch(p, fam.hierarchy[1], PararealConfig(4, 1e-4, 1e-3, 1e-8, 4))


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    name = sys.argv[1]
    globals()["case_" + name]()
    torch.cuda.synchronize()
    print(f"{name} ok", flush=True)
