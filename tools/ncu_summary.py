"""Summarise an ncu report: key metrics per kernel + top SASS lines by instructions/stalls."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_op_red.sum", "lts__t_requests_op_red.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
idx = {w: hdr.index(w) for w in want if w in hdr}
for r in rows[2:]:
    print("----")
    for w, i in idx.items():
        print(f"  {w:60s} {r[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; kernels.append(cur); continue
    if cur is None: continue
    if r and r[0] == "Address": cur["hdr"] = r; continue
    cur["rows"].append(r)
seen = set()
for k in kernels:
    if k["name"] in seen: continue
    seen.add(k["name"])
    h = k["hdr"]; ie = h.index("Instructions Executed"); st = h.index("Warp Stall Sampling (All Samples)")
    out = [(int(r[ie]), int(r[st]), r[1].strip()) for r in k["rows"] if len(r) > ie and r[ie].isdigit()]
    tot = sum(x[0] for x in out); tots = max(1, sum(x[1] for x in out))
    print(f"===== {k['name'][:90]}  inst {tot}  samples {tots}")
    sel = sorted(range(len(out)), key=lambda j: -(out[j][0] / max(tot, 1) + out[j][1] / tots))[:top]
    for j in sorted(sel):
        n, s_, src_ = out[j]
        print(f"{j:5d} {n:>11} {100*n/max(tot,1):5.1f}% st{100*s_/tots:5.1f}%  {src_}")
