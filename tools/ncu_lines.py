"""Top CUDA source lines of one ncu report (--import-source, -lineinfo) by warp-stall samples."""
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = lambda v: float(v) if v.replace('.', '', 1).isdigit() else 0.0
hdr, fname, func, res = None, None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split('/')[-1]
    elif r and r[0] == "Function Name":
        func = r[1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 4 and r[0].isdigit() and r[2] == "-":
        if kfilter is None or kfilter in (func or ""):
            res.append((fname, int(r[0]), r[1], f(r[4]), r))
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(x[3] for x in res) or 1
for fl, ln, src, s, r in sorted(res, key=lambda x: -x[3])[:top]:
    rs = sorted(((f(r[i]), h[6:]) for i, h in reasons), reverse=True)[:3]
    print(f"{s / tot * 100:5.1f}% {fl}:{ln} {src.strip()[:64]:64s} " + " ".join(f"{h}:{v:.0f}" for v, h in rs if v))
