"""A/B of the streaming-path implementations on one batch: the cluster kernel
(MLMCP_STREAM_IMPL=3, one thread-block cluster per task) against the two-launch
HBM-streaming kernels (=1) — QoIs, terminal states, PCG iterations and time.
    python scripts/cluster_check.py [CFG S STEPS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2507_19246_b200.mlmc import draw_level
from paper_2507_19246_b200.models import eddy_current_family


def run(fam, M, K, S, steps, impl, reps=2):
    os.environ["MLMCP_STREAM_IMPL"] = str(impl)
    sol = fam.solver
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
    x = sol._last_xbuf.view(S, -1).clone()
    return res, x, float(np.median(times))


def main(cfg=3, S=64, steps=16):
    fam = eddy_current_family(cfg, device="cuda:0")
    sol = fam.solver
    p = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
    M, K = sol.assemble(torch.from_numpy(p).cuda())
    b_it = 8 * sol.mesh.nnz + 56 * sol.N
    out = {}
    for impl in (1, 3):
        res, x, s = run(fam, M, K, S, steps, impl)
        its = int(res.iters.to(torch.int64).sum().item())
        st = int(res.status[:, 0].abs().sum().item())
        out[impl] = (res.qoi.double().cpu().numpy(), x.cpu().numpy())
        print(f"impl={impl} cfg{cfg} N={sol.N} S={S} steps={steps}: its={its} "
              f"({its / S / steps:.2f}/step) time={s * 1e3:.2f} ms  status_sum={st}  "
              f"{its / s / 1e6:.2f} M sample-its/s  (algorithmic {its * b_it / s / 1e9:.0f} GB/s)",
              flush=True)
    q1, x1 = out[1]
    q3, x3 = out[3]
    rq = np.max(np.abs(q3 - q1) / np.abs(q1))
    rx = np.max(np.abs(x3 - x1)) / np.max(np.abs(x1))
    print(f"max rel QoI diff {rq:.3e}, max state diff / max|x| {rx:.3e}")


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
