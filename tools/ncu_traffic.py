"""Summarise an ncu --set full capture of one admm_persistent launch (tools/prof_admm.py) into
profiles/ncu_admm_traffic.json: DRAM bytes per launch vs the launch's algorithmic bytes, plus the
headline metrics (developer tool; bench.py reads the ratio for roofline.traffic).
    python tools/ncu_traffic.py gpurun_out/admm_full.ncu-rep <iters> <nb> <n> <p> "<capture description>"
"""
import csv
import io
import json
import subprocess
import sys

rep, iters, nb, n, p, desc = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(name, scale={"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}):
    v, u = m[name]
    return float(v.replace(",", "")) * scale.get(u, 1)


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
# algorithmic bytes of the launch: per iteration (+ the refresh sweep) one read
# of Z (8np) and the node state (33p per node)
alg = (iters + 1) * (8.0 * n * p + 33.0 * p * nb)
keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]
d = {"capture": desc, "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
     "alg_bytes_per_launch": alg, "dram_bytes_per_launch_per_alg_byte": (rd + wr) / alg,
     "why_above_1": "per launch: +1 forward-only sweep for u0 (amortised over the launch's iterations); with "
                    "16 nodes the two CTAs of a pair stream the same tiles and the second read is an L2 hit "
                    "only when the pair stays in step; the u reduction partials and the sparse primal "
                    "check's X gathers (β⁺ nonzeros only) are small",
     "metrics": {k: list(m[k][::-1])[::-1] if False else [m[k][0], m[k][1]] for k in keep if k in m}}
json.dump(d, open("profiles/ncu_admm_traffic.json", "w"), indent=1)
print(json.dumps({k: d[k] for k in ("dram_bytes_per_launch", "alg_bytes_per_launch", "dram_bytes_per_launch_per_alg_byte")}))
