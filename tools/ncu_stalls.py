"""Stall-reason breakdown, occupancy limits and per-region SASS instruction shares of an ncu report."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for v in rows[2:]:
    d = {h[i]: v[i] for i in range(len(h))}
    print("====", d.get("Kernel Name", "")[:80])
    st = []
    for k, x in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((k[33:], float(x)))
            except ValueError:
                pass
    tot = sum(x for _, x in st) or 1
    for k, x in sorted(st, key=lambda a: -a[1])[:10]:
        print(f"  stall {k:40s} {100 * x / tot:5.1f}%")
    for k in ["sm__warps_active.avg.per_cycle_active", "launch__occupancy_limit_shared_mem",
              "launch__occupancy_limit_registers", "launch__registers_per_thread", "launch__grid_size",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]:
        print(f"  {k:55s} {d.get(k)}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
out, hdr = [], None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        if out:
            break
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) > 5:
        ie, sti = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        if r[ie].isdigit():
            out.append((int(r[ie]), int(r[sti]), r[1].strip()))
tot = sum(x[0] for x in out) or 1
ts = sum(x[1] for x in out) or 1
print("==== SASS regions (25 lines each) with >0.5% of instructions or stalls")
for b in range(0, len(out), 25):
    blk = out[b:b + 25]
    n, s = sum(x[0] for x in blk), sum(x[1] for x in blk)
    if n / tot > 0.005 or s / ts > 0.005:
        print(f"  {b:5d} inst {100 * n / tot:5.1f}% stall {100 * s / ts:5.1f}%  x{blk[0][0]:<10d} {blk[0][2][:60]}")
