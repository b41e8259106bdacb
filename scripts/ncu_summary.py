"""Summarise an ncu --set full report into a JSON under profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.json [--top]
--top also writes profiles/ncu_top_kernel.json (read by bench.py for
roofline.traffic = dram bytes read + written per launch)."""
import csv
import json
import subprocess
import sys

KEEP = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed")


def main(rep, out, top=False):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")][:120]}
        stalls = {}
        for i, n in enumerate(hdr):
            if n in KEEP:
                d[n] = {"value": v[i], "unit": units[i]}
            if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]) if x}
        def num(key, scale):
            x = d.get(key)
            if x is None:
                return None
            f = float(x["value"].replace(",", ""))
            u = x["unit"].lower()
            mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-9,
                    "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6,
                    "ms": 1e-3, "s": 1}.get(u, 1)
            return f * mult / scale
        rd, wr = num("dram__bytes_read.sum", 1), num("dram__bytes_write.sum", 1)
        d["dram_bytes_per_launch"] = (rd or 0) + (wr or 0)
        d["duration_s"] = num("gpu__time_duration.sum", 1)
        kernels.append(d)
    json.dump({"report": rep, "kernels": kernels}, open(out, "w"), indent=1)
    if top:
        k = kernels[0]
        json.dump({"kernel": k["kernel"], "dram_bytes_per_launch": k["dram_bytes_per_launch"],
                   "duration_s": k["duration_s"], "source": out},
                  open("profiles/ncu_top_kernel.json", "w"), indent=1)
    print(json.dumps(kernels[0], indent=1)[:2000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], "--top" in sys.argv)
