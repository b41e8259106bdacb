"""A/B of the streaming tile path on a config-2 / config-4 level-0 batch:
streamed operator ([S][4][N] symmetric halves, MLMCP_TILE_OPERATOR=stored)
vs the region-linear operator computed in the kernels (default).
Prints one JSON line per mode: propagate-call time, PCG-iteration launch time
(CUDA events inside libmlmcp), iterations, achieved GB/s against B_it and
against the bytes the mode actually streams.
Modes: stored, region (recompute-w kernel, 64 B/point), regionw (stored-w
region kernel, 80 B/point), band (cluster-resident band path, 256^2 grids);
"@n" appends MLMCP_TILE_CFG=n.
usage: python scripts/tile_ab.py [CFG=2] [S=1024] [STEPS=32] [MODES]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_19246_b200.configs import get_config  # noqa: E402
from paper_2507_19246_b200.mlmc import draw_level  # noqa: E402
from paper_2507_19246_b200.models import eddy_current_family  # noqa: E402

cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
modes = sys.argv[4].split(",") if len(sys.argv) > 4 else ["stored", "region"]
peak = 6443.2
try:
    peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
cfg = get_config(cfg_i)
qs = {}
for mode in modes:
    op, _, tcfg = mode.partition("@")       # e.g. "region@3": MLMCP_TILE_CFG=3
    rw = op != "regionw"                    # "regionw": region operator, stored-w kernel
    os.environ["MLMCP_TILE_RW"] = "1" if rw else "0"
    os.environ["MLMCP_BAND"] = "1" if op == "band" else "0"   # "band": 16-CTA cluster path
    op = "region" if op in ("regionw", "band") else op
    os.environ["MLMCP_TILE_OPERATOR"] = op
    if tcfg:
        os.environ["MLMCP_TILE_CFG"] = tcfg
    else:
        os.environ.pop("MLMCP_TILE_CFG", None)
    fam = eddy_current_family(cfg_i, device="cuda:0")
    sol = fam.solver
    d = draw_level(fam.uncertain, 0, 0, range(1, S + 1))
    pd = torch.from_numpy(d).cuda()
    M = torch.empty((S, sol.nnz), dtype=torch.float64, device="cuda")
    K = torch.empty_like(M)
    rp = sol.new_region_params(S)
    sol.assemble(pd, out=(M, K), rp_out=rp)
    job = fam._seq_job(np.arange(S), fam.hierarchy[int(os.environ.get("TILE_AB_LEVEL", "0"))].dt)
    job.n_steps = steps
    times = []
    for r in range(3):
        if r == 1:
            sol.sys.stream_timing(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = sol.run_sequential(M, K, [job], rp=rp)[0]
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    it_ms, launches = sol.sys.stream_timing(0)
    its = int(res.iters.to(torch.int64).sum().item())
    b_it = 8 * sol.nnz + 56 * sol.N
    actual = ((64 if rw else 80) if sol.region_mode else 112) * sol.N
    k_ms = it_ms / 2 if it_ms > 0 else float(np.mean(times))   # band path: no iteration launches
    qs[mode] = res.qoi.cpu().numpy()
    print(json.dumps({"mode": mode, "region": sol.region_mode, "cfg": cfg_i, "S": S, "steps": steps,
                      "call_ms": float(np.mean(times)), "iter_kernel_ms": k_ms,
                      "iter_launches": launches // 2, "pcg_iterations": its,
                      "its_per_step": its / (S * steps),
                      "achieved_B_it_gbs": its * b_it / (k_ms / 1e3) / 1e9,
                      "frac_B_it": its * b_it / (k_ms / 1e3) / 1e9 / peak,
                      "achieved_actual_gbs": its * actual / (k_ms / 1e3) / 1e9,
                      "frac_actual": its * actual / (k_ms / 1e3) / 1e9 / peak,
                      "call_frac_B_it": its * b_it / (np.mean(times) / 1e3) / 1e9 / peak}),
          flush=True)
    del M, K, rp, res, fam, sol
    torch.cuda.empty_cache()
if len(qs) >= 2:
    vals = list(qs.values())
    a = vals[0]
    for name, b in list(qs.items())[1:]:
        print(json.dumps({"vs_first": name,
                          "max_rel_qoi_diff": float(np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300))),
                          "bitwise": bool(np.array_equal(a, b))}))
