"""One-line-per-kernel brief of an ncu report: duration, DRAM/L2/SM throughput,
occupancy, and the top warp-stall reasons.  usage: python tools/ncu_brief.py REP"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]


units = dict(zip(hdr, rows[1]))
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
         "Gbyte": 1e3, "%": 1.0}


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return 0.0


def val(d, k):
    return num(d[k]) * SCALE.get(units.get(k, ""), 1.0)


want = {"gpu__time_duration.sum": "us", "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
        "lts__t_sectors_op_read.sum": "l2rd_sect", "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
        "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
        "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active": "tc%"}
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("_not_issued")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    parts = [d.get("Kernel Name", "")[:34].ljust(34), d.get("Grid Size", ""), d.get("Block Size", "")]
    for k, nm in want.items():
        if k in d:
            parts.append(f"{nm}={val(d, k):.1f}")
    st = sorted(((num(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, h in stall_cols),
                reverse=True)
    tot = sum(v for v, _ in st) or 1.0
    parts.append(" ".join(f"{h}:{100 * v / tot:.0f}%" for v, h in st[:4]))
    print(" ".join(parts))
