"""Group consecutive SASS lines of one kernel with equal execution counts (basic blocks)."""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; kernels.append(cur); continue
    if cur is None: continue
    if r and r[0] == "Address": cur["hdr"] = r; continue
    cur["rows"].append(r)
k = [k for k in kernels if pat in k["name"]][0]
h = k["hdr"]; ie = h.index("Instructions Executed"); te = h.index("Thread Instructions Executed")
st = h.index("Warp Stall Sampling (All Samples)")
out = [(int(r[ie]), int(r[te]), int(r[st]), r[1].strip()) for r in k["rows"] if len(r) > ie and r[ie].isdigit()]
tot = sum(x[0] for x in out); tots = max(1, sum(x[2] for x in out))
groups = []
for i, (n, t, s_, src_) in enumerate(out):
    if groups and groups[-1]["n"] == n:
        g = groups[-1]; g["c"] += 1; g["t"] += t; g["s"] += s_; g["last"] = src_
    else:
        groups.append({"n": n, "c": 1, "t": t, "s": s_, "first": src_, "last": src_, "i": i})
print(f"{k['name'][:100]}\ntotal inst {tot}")
for g in groups:
    if g["n"] * g["c"] > thr * tot or g["s"] > 0.03 * tots:
        print(f"@{g['i']:4d} {g['n']:>10} x{g['c']:3d} = {100*g['n']*g['c']/tot:5.1f}%  stall {100*g['s']/tots:5.1f}%  thr/inst {g['t']/max(1,g['n']*g['c']):5.1f}  {g['first'][:45]} .. {g['last'][:35]}")
