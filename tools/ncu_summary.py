"""Summarise an ncu --set full capture of one admm_persistent launch whose algorithmic bytes / flops
are known (e.g. a tree-step launch: tools/ncu_tree_step.py difference of two node limits) into a JSON
file (developer tool; bench.py reads dram_bytes_per_launch_per_alg_byte for roofline.traffic).
    python tools/ncu_summary.py REP ALG_BYTES ALG_FLOPS OUT.json "<capture description>" """
import csv
import io
import json
import subprocess
import sys

rep, alg, algf, outp, desc = sys.argv[1], float(sys.argv[2]), float(sys.argv[3]), sys.argv[4], sys.argv[5]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
      "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "s": 1.0, "second": 1.0}


def num(name):
    v, u = m[name]
    return float(v.replace(",", "")) * SC.get(u, 1)


rd, wr, t = num("dram__bytes_read.sum"), num("dram__bytes_write.sum"), num("gpu__time_duration.sum")
keep = [k for k in m if any(s in k for s in (
    "gpu__time_duration.sum", "dram__bytes", "dmma", "sm__warps_active.avg.pct", "lts__t_sector_hit_rate.pct",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "l1tex__m_xbar2l1tex_read_bytes",
    "sm__throughput.avg.pct", "gpu__compute_memory_throughput.avg.pct"))]
d = {"capture": desc, "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
     "alg_bytes_per_launch": alg, "alg_flops_per_launch": algf, "dram_bytes_per_launch_per_alg_byte": (rd + wr) / alg,
     "ncu_time_s": t, "alg_tflops_under_ncu": algf / t / 1e12, "dram_tbs_under_ncu": (rd + wr) / t / 1e12,
     "metrics": {k: [m[k][0], m[k][1]] for k in sorted(keep)}}
json.dump(d, open(outp, "w"), indent=1)
print(json.dumps({k: d[k] for k in ("dram_bytes_per_launch", "alg_bytes_per_launch", "dram_bytes_per_launch_per_alg_byte",
                                     "ncu_time_s", "alg_tflops_under_ncu")}))
