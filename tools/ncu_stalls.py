"""Top SASS lines of one ncu report by warp-stall samples, with their dominant stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
f = lambda v: float(v) if v and v.replace('.', '', 1).isdigit() else 0.0
i_s = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(f(r[i_s]) for r in data) or 1
for r in sorted(data, key=lambda r: -f(r[i_s]))[:top]:
    rs = sorted(((f(r[i]), h[6:]) for i, h in reasons), reverse=True)[:3]
    print(f"{f(r[i_s]) / tot * 100:5.1f}% {r[0][-5:]} {r[1][:60]:60s} " + " ".join(f"{h}:{v:.0f}" for v, h in rs if v))
