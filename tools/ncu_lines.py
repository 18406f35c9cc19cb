"""Per CUDA source line: instructions executed and stall samples of one kernel in an ncu report
(needs -lineinfo and --import-source on).  usage: ncu_lines.py rep.ncu-rep FUNC_SUBSTR [top]"""
import csv, io, subprocess, sys

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fpath, func, hdr, out, done = None, None, None, [], False
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        func = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if func is None or ksub not in func or not r[0].isdigit():
        continue
    ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    n = int(r[ie]) if r[ie].isdigit() else 0
    s = int(r[st]) if r[st].isdigit() else 0
    if n or s:
        out.append((fpath, int(r[0]), r[1].strip()[:100], n, s))
tot = sum(o[3] for o in out) or 1
tots = sum(o[4] for o in out) or 1
print(f"{ksub}  inst {tot}  samples {tots}")
sel = sorted(out, key=lambda o: -(o[3] / tot + o[4] / tots))[:top]
for f, ln, s_, n, s in sorted(sel, key=lambda o: (o[0], o[1])):
    print(f"{100*n/tot:5.1f}% {100*s/tots:5.1f}%  {f}:{ln:<5d} {s_}")
