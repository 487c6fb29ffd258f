"""Print the top stall lines of one kernel from an ncu report (SASS view)."""
import csv
import subprocess
import sys

rep, regex, skip = sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{regex}", "--launch-skip", str(skip),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
f = lambda v: float(v) if v else 0.0
tot = sum(f(r[i_s]) for r in data) or 1
print("kernel:", rows[0][1] if len(rows[0]) > 1 else rows[0])
for r in sorted(data, key=lambda r: -f(r[i_s]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    print(f"{f(r[i_s]) / tot * 100:5.1f}%  {r[0][-5:]} {r[i_src][:100]}")
