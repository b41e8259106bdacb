"""Summarise one kernel launch of an ncu --set full capture into the JSON the
bench reads (profiles/ncu_top_kernel.json): dram bytes per launch and per PCG
task-iteration next to the algorithmic figures.
usage: python scripts/ncu_summary.py REPORT.ncu-rep KEY TASK_ITERATIONS POINTS NNZ BYTES_PER_POINT OUT.json [LAUNCH_DESC]"""
import csv
import json
import subprocess
import sys


def main():
    rep, key, tasks, pts, nnz, bpp, out = sys.argv[1:8]
    desc = sys.argv[8] if len(sys.argv) > 8 else ""
    tasks, pts, nnz, bpp = int(tasks), int(pts), int(nnz), int(bpp)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader([ln for ln in txt.splitlines() if ln.startswith('"')]))
    d = {h: (v, u) for h, u, v in zip(*r[:3])}

    def g(k):
        v, u = d[k]
        v = float(v.replace(",", ""))
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(u, 1.0)
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    ms = g("gpu__time_duration.sum") * (1e-3 if d["gpu__time_duration.sum"][1] == "us" else 1.0)
    b_it = 8 * nnz + 56 * pts
    ent = {"kernel": d["Kernel Name"][0], "source": out, "launch": desc, "duration_ms": ms,
           "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
           "dram_gbs": (rd + wr) / (ms * 1e-3) / 1e9, "task_iterations_per_launch": tasks,
           "dram_bytes_per_task_iteration": (rd + wr) / tasks,
           "algorithmic_bytes_per_task_iteration_B_it": b_it,
           "streamed_bytes_per_task_iteration": bpp * pts,
           "algorithmic_bytes_per_launch": tasks * b_it,
           "sm_throughput_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
           "issue_slots_busy_pct": g("sm__inst_issued.avg.pct_of_peak_sustained_active"),
           "ipc_active": g("sm__inst_executed.avg.per_cycle_active"),
           "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
           if "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" in d else None,
           "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
           "registers": int(g("launch__registers_per_thread"))}
    with open(out, "w") as fh:
        json.dump(ent, fh, indent=1)
    top = "profiles/ncu_top_kernel.json"
    try:
        allk = json.load(open(top))
        if "kernel" in allk:          # old flat format
            allk = {}
    except Exception:
        allk = {}
    allk[key] = ent
    with open(top, "w") as fh:
        json.dump(allk, fh, indent=1)
    print(json.dumps(ent, indent=1))


if __name__ == "__main__":
    main()
