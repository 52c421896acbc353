"""Summarise an ncu report: key metrics, stall reasons, and top SASS lines by stall samples."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__thread_inst_executed_op_dfma_pred_on.sum"]
for h, u, v in zip(hdr, units, vals):
    if h in want:
        print(f"{h:70s} {v:>18s} {u}")
stalls = [(h, v) for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and
          not h.endswith("_not_issued")]
tot = sum(float(v) for _, v in stalls if v)
for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:10]:
    print(f"  stall {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {float(v) / tot * 100:5.1f}%")
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
h2 = src[1]
data = src[2:]
iss = h2.index("Warp Stall Sampling (All Samples)")
iex = h2.index("Instructions Executed")
isrc = h2.index("Source")
c, s = Counter(), Counter()
for r in data:
    parts = r[isrc].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    op = op.split(".")[0]
    c[op] += int(r[iex] or 0)
    s[op] += int(r[iss] or 0)
tot_i = sum(c.values())
tot_s = sum(s.values())
print("instructions", tot_i)
for op, v in c.most_common(18):
    print(f"  {op:10s} {v / tot_i * 100:5.1f}% inst  {s[op] / max(tot_s, 1) * 100:5.1f}% stall")
data.sort(key=lambda r: -int(r[iss] or 0))
print("top stall lines")
for r in data[:top]:
    print(f"  {int(r[iss]) / max(tot_s, 1) * 100:5.1f}%  {r[0][-5:]}  {r[isrc][:70]}")

# per CUDA source line (needs -lineinfo)
try:
    src2 = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "cuda"]))))
    h3 = src2[1] if len(src2) > 1 else []
    if "Warp Stall Sampling (All Samples)" in h3:
        i_s = h3.index("Warp Stall Sampling (All Samples)")
        i_l = h3.index("Line") if "Line" in h3 else 0
        i_src = h3.index("Source")
        rows = [r for r in src2[2:] if len(r) > i_s and r[i_s]]
        tot3 = sum(int(r[i_s]) for r in rows) or 1
        rows.sort(key=lambda r: -int(r[i_s]))
        print("top CUDA lines by stall samples")
        for r in rows[:top]:
            print(f"  {int(r[i_s]) / tot3 * 100:5.1f}%  L{r[i_l]:>5s}  {r[i_src].strip()[:90]}")
except Exception as ex:  # older ncu: no cuda view
    print("no CUDA-line view:", ex)
