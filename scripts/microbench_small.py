"""Micro-benchmark of the SM-resident propagate kernel: S samples of the 32x32
config-1 mesh, n_steps implicit-Euler steps at dt = T/256, one launch.
Prints PCG iterations, kernel ms and cycles per PCG iteration per SM slot."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2507_19246_b200.configs import T
from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family


def main(S=296 * 2, steps=64, reps=3):
    fam = eddy_current_family(1, device="cuda:0")
    sol = fam.solver
    p = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
    M, K = sol.assemble(torch.from_numpy(p).cuda())
    job = fam._seq_job(np.arange(S), T / 256)
    job.n_steps = steps
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    sol.events = ev
    out = []
    for r in range(reps + 1):
        res = sol.run_sequential(M, K, [job])[0]
        torch.cuda.synchronize()
        if r:
            out.append(ev[0].elapsed_time(ev[1]))
    its = int(res.iters.to(torch.int64).sum().item())
    ms = float(np.median(out))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk = 1.965e9
    print(f"S={S} steps={steps} its={its} ({its / S / steps:.1f}/step) kernel={ms:.3f} ms "
          f"-> {ms * 1e-3 * clk * sms / its:.0f} SM-cycles per PCG iteration "
          f"(OCC env {os.environ.get('MLMCP_SMALL_OCC', 'default')})")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
