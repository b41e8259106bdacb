"""Micro-benchmark of the HBM-streaming path (meshes > 1024 rows): S samples of
config C's mesh, n_steps implicit-Euler steps at the config's level-0 dt, one
propagate call.  Prints PCG iterations and the achieved algorithmic bandwidth
B_it = 8 nnz + 56 N bytes per PCG iteration per sample."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family


def main(cfg=3, S=256, steps=16, reps=2):
    fam = eddy_current_family(cfg, device="cuda:0")
    sol = fam.solver
    p = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
    M, K = sol.assemble(torch.from_numpy(p).cuda())
    dt = fam.hierarchy[0].dt
    job = fam._seq_job(np.arange(S), dt)
    job.n_steps = steps
    times = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = sol.run_sequential(M, K, [job])[0]
        torch.cuda.synchronize()
        if r:
            times.append(time.perf_counter() - t)
    its = int(res.iters.to(torch.int64).sum().item())
    s = float(np.median(times))
    b_it = 8 * sol.mesh.nnz + 56 * sol.N
    print(f"cfg{cfg} n={sol.n} N={sol.N} S={S} steps={steps}: its={its} ({its / S / steps:.1f}/step) "
          f"time={s * 1e3:.1f} ms  algorithmic {its * b_it / s / 1e9:.0f} GB/s "
          f"({its / S / s:.0f} its/s/sample)")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
