"""Summarise this round's ncu evidence into profiles/ (committed):
  profiles/ncu_launches_<tag>.csv   the launch list of one bench step (dyn + dense)
  profiles/ncu_full_<tag>.json      per-kernel metrics of the --set full capture
  profiles/ncu_summary_<tag>.md     human-readable table
Usage: python tools/ncu_summary.py <tag>   (reads gpurun_out/launches_<tag>.csv, full_<tag>.ncu-rep)
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)


def short(name):
    name = name.replace("lasnet::", "").replace("(lasnet::ConvArgs)", "")
    table = {"conv_tc_kernel<0,": "conv1_dyn", "conv_tc_kernel<1,": "conv2_dyn", "conv_tc_kernel<2,": "conv3_dyn",
             "conv_tc_kernel<3,": "conv1_dense", "conv_tc_kernel<4,": "conv2_dense", "conv_tc_kernel<5,": "conv3_dense",
             "conv23_kernel<(bool)0>": "conv23_dyn", "conv23_kernel<(bool)1>": "conv23_dense",
             "conv23_kernel<0>": "conv23_dyn", "conv23_kernel<1>": "conv23_dense",
             "conv23_kernel<false>": "conv23_dyn", "conv23_kernel<true>": "conv23_dense",
             "masker_compact_kernel": "mask_compact", "masker_kernel": "mask", "compact_kernel": "compact"}
    flat = name.replace(" ", "").replace("(int)", "")
    for k, v in table.items():
        if k.replace(" ", "") in flat:
            return v
    return name[:40]


# ---------------------------------------------------------- launch list ----
lines = open(os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(lines[start:]))
per = {}
for r in rows:
    per.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
    per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
launches = [dict(id=int(k), kernel=short(v["name"]), grid=v["grid"], block=v["block"],
                 time_ns=v.get("gpu__time_duration.sum"), dram_read=v.get("dram__bytes_read.sum"),
                 dram_write=v.get("dram__bytes_write.sum")) for k, v in per.items()]
launches.sort(key=lambda d: d["id"])
# the last dynamic step: last mask_compact and the three convs after it
DYN = ("conv1_dyn", "conv2_dyn", "conv3_dyn", "conv23_dyn")
DENSE = ("conv2_dense", "conv3_dense", "conv23_dense")
idx_mc = max(i for i, d in enumerate(launches) if d["kernel"] == "mask_compact")
step = [launches[idx_mc]]
for d in launches[idx_mc + 1:]:
    if d["kernel"] not in DYN:
        break
    step.append(d)
dense_ids = [i for i, d in enumerate(launches) if d["kernel"] == "conv1_dense"]
dense = []
if dense_ids:
    dense = [launches[dense_ids[-1]]]
    for d in launches[dense_ids[-1] + 1:]:
        if d["kernel"] not in DENSE:
            break
        dense.append(d)
with open(os.path.join(out_dir, f"ncu_launches_{tag}.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "time_ns", "dram_read_bytes", "dram_write_bytes"])
    for d in launches:
        w.writerow([d["id"], d["kernel"], d["grid"], d["block"], d["time_ns"], d["dram_read"], d["dram_write"]])

# ----------------------------------------------------------- full capture ---
rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hdr = rr[0]
want = {
    "time_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
}
units = rr[1]
full = []
for r in rr[2:]:
    d = {"kernel": short(r[hdr.index("Kernel Name")])}
    for k, m in want.items():
        if m in hdr:
            v = r[hdr.index(m)].replace(",", "")
            try:
                d[k] = float(v)
            except ValueError:
                d[k] = v
            u = units[hdr.index(m)]
            if k == "time_ns" and u in ("usecond", "us"):
                d[k] *= 1e3
            if k.startswith("dram_r") or k.startswith("dram_w"):
                if u == "Mbyte":
                    d[k] *= 1e6
                elif u == "Kbyte":
                    d[k] *= 1e3
                elif u == "Gbyte":
                    d[k] *= 1e9
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), r[i]) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    st = [(h, float(v.replace(",", ""))) for h, v in st if v]
    tot = sum(v for _, v in st) or 1.0
    d["top_stalls"] = {h: round(v / tot, 3) for h, v in sorted(st, key=lambda x: -x[1])[:4]}
    full.append(d)
json.dump({"tag": tag, "step_launches": step, "dense_launches": dense, "full": full},
          open(os.path.join(out_dir, f"ncu_full_{tag}.json"), "w"), indent=1)

# --------------------------------------------------------------- summary ----
md = [f"# ncu summary ({tag})", "",
      "Source: `tools/prof_round.sh " + tag + "` on one B200 (gpurun). Launch list: "
      "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` "
      "(cold-cache, serialised: compare shares, not absolutes). Full capture: `ncu --set full --clock-control none`.",
      "", "## One dynamic step (bench workload: N=128, 28x28x512, c_mid=128, S=4, r~0.5)", "",
      "| kernel | grid x block | time (us) | share | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|---|"]
tot = sum(d["time_ns"] or 0 for d in step) or 1
for d in step:
    md.append(f"| {d['kernel']} | {d['grid']} x {d['block']} | {d['time_ns'] / 1e3:.1f} | "
              f"{(d['time_ns'] or 0) / tot:.2f} | {(d['dram_read'] or 0) / 1e6:.1f} | {(d['dram_write'] or 0) / 1e6:.1f} |")
md.append(f"| **total** | | **{tot / 1e3:.1f}** | | | |")
if dense:
    md += ["", "## Dense comparator (lasnet_dense_block, same shapes)", "",
           "| kernel | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|"]
    for d in dense:
        md.append(f"| {d['kernel']} | {d['time_ns'] / 1e3:.1f} | {(d['dram_read'] or 0) / 1e6:.1f} | "
                  f"{(d['dram_write'] or 0) / 1e6:.1f} |")
md += ["", "## Full capture (per kernel)", "",
       "| kernel | time (us) | DRAM rd+wr (MB) | DRAM % | tensor % | SM % | L2 % | warps active % | regs | top stalls |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for d in full:
    md.append(f"| {d['kernel']} | {d.get('time_ns', 0) / 1e3:.1f} | "
              f"{(d.get('dram_read', 0) + d.get('dram_write', 0)) / 1e6:.1f} | {d.get('dram_pct', 0):.1f} | "
              f"{d.get('tensor_pct', 0):.1f} | {d.get('sm_pct', 0):.1f} | {d.get('l2_pct', 0):.1f} | "
              f"{d.get('warps_active_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
              + ", ".join(f"{k} {v:.0%}" for k, v in d["top_stalls"].items()) + " |")
open(os.path.join(out_dir, f"ncu_summary_{tag}.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
