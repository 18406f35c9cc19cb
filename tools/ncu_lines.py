"""Per CUDA-source-line instruction counts and stall samples of one kernel in an ncu report
(needs -lineinfo).  usage: ncu_lines.py report.ncu-rep [kernel-substring] [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows, cur, hdr, want = [], None, None, False
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        want = ksub in r[1] and cur is None
        if want:
            cur = r[1]
        continue
    if not want:
        continue
    if r and r[0] in ("#", "Line", "Address"):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rows.append(dict(zip(hdr, r)))
if not rows:
    print("no rows; headers:", hdr)
    sys.exit()
ik = [k for k in rows[0] if k.startswith("Instructions Executed")][0]
sk = [k for k in rows[0] if k.startswith("Warp Stall Sampling (All")][0]
src = [k for k in rows[0] if k == "Source"][0]
num = lambda x: float(x) if x.replace(".", "").isdigit() else 0.0
tot_i = sum(num(r[ik]) for r in rows) or 1
tot_s = sum(num(r[sk]) for r in rows) or 1
print(f"kernel {cur[:100]}\ninstructions {tot_i:.3e}  stall samples {tot_s:.0f}")
sel = sorted(rows, key=lambda r: -(num(r[ik]) / tot_i + num(r[sk]) / tot_s))[:top]
for r in sorted(sel, key=lambda r: int(r.get("#", r.get("Line", "0")) or 0)):
    ln = r.get("#", r.get("Line", ""))
    print(f"{ln:>5} inst {100 * num(r[ik]) / tot_i:5.1f}% stall {100 * num(r[sk]) / tot_s:5.1f}%  {r[src].strip()[:100]}")
