"""Summarise one round's ncu evidence for BOTH schedules into profiles/ (committed).

Inputs (written by tools/prof_r1c.sh TAG into gpurun_out/):
  launches_<tag>.csv, launches_<tag>_sep.csv   launch lists of the bench command (fused / separate schedule)
  full_<tag>.ncu-rep, full_<tag>_sep.ncu-rep   --set full captures of each kernel
Outputs:
  profiles/ncu_launches_<tag>.csv   both launch lists (schedule column)
  profiles/ncu_full_<tag>.json      per-kernel metrics (bench.py reads DRAM traffic from here)
  profiles/ncu_summary_<tag>.md     tables
usage: python tools/ncu_summary2.py <tag>
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1c"
OUT = os.path.join(ROOT, "profiles")
GO = os.path.join(ROOT, "gpurun_out")


def short(name):
    n = name.replace("lasnet::", "").replace(" ", "").replace("(int)", "").replace("(bool)", "")
    table = [("conv_tc_kernel<0,", "conv1_dyn"), ("conv_tc_kernel<1,", "conv2_dyn"), ("conv_tc_kernel<2,", "conv3_dyn"),
             ("conv_tc_kernel<3,", "conv1_dense"), ("conv_tc_kernel<4,", "conv2_dense"),
             ("conv_tc_kernel<5,", "conv3_dense"), ("conv_tc_kernel<6,", "conv1_mask"),
             ("conv23_kernel<0", "conv23_dyn"), ("conv23_kernel<false", "conv23_dyn"),
             ("conv23_kernel<1", "conv23_dense"), ("conv23_kernel<true", "conv23_dense"),
             ("masker_compact_kernel", "mask_compact"), ("masker_kernel", "mask"), ("compact_kernel", "compact"),
             ("decide_kernel", "decide"), ("compact_gather_kernel", "compact_gather"),
             ("compact_idx_kernel", "compact_idx")]
    for k, v in table:
        if k in n:
            return v
    return name[:40]


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    per = {}
    for r in csv.DictReader(lines[start:]):
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    out = [dict(id=int(k), kernel=short(v["name"]), grid=v["grid"], block=v["block"],
                time_ns=v.get("gpu__time_duration.sum"), dram_read=v.get("dram__bytes_read.sum"),
                dram_write=v.get("dram__bytes_write.sum")) for k, v in per.items()]
    return sorted(out, key=lambda d: d["id"])


def last_step(ls, first, members):
    i0 = max(i for i, d in enumerate(ls) if d["kernel"] == first)
    step = [ls[i0]]
    for d in ls[i0 + 1:]:
        if d["kernel"] not in members:
            break
        step.append(d)
    return step


WANT = {
    "time_ns": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_tex_sectors": "lts__t_sectors_srcunit_tex.sum",
    "smem_lsu_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_tc_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
}
SCALE = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr, units = rr[0], rr[1]
    res = []
    for r in rr[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, m in WANT.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), r[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        st = [(h, float(v.replace(",", ""))) for h, v in st if v]
        tot = sum(v for _, v in st) or 1.0
        d["top_stalls"] = {h: round(v / tot, 3) for h, v in sorted(st, key=lambda x: -x[1])[:3]}
        res.append(d)
    return res


lf = launches(os.path.join(GO, f"launches_{tag}.csv"))
lsep = launches(os.path.join(GO, f"launches_{tag}_sep.csv"))
step_f = last_step(lf, "conv1_mask", ("decide", "compact_gather", "compact_idx", "conv23_dyn", "conv2_dyn", "conv3_dyn"))
step_s = last_step(lsep, "mask_compact", ("conv1_dyn", "conv23_dyn", "conv2_dyn", "conv3_dyn"))
dense = last_step(lf, "conv1_dense", ("conv23_dense", "conv2_dense", "conv3_dense"))
full_f = full(os.path.join(GO, f"full_{tag}.ncu-rep"))
full_s = full(os.path.join(GO, f"full_{tag}_sep.ncu-rep")) if os.path.exists(os.path.join(GO, f"full_{tag}_sep.ncu-rep")) else []
# one entry per kernel (first capture), plus the combined decide+gather launch pair bench.py reports
fullk = {}
for d in full_f + full_s:
    fullk.setdefault(d["kernel"], d)
second = "compact_gather" if "compact_gather" in fullk else "compact_idx"
if "decide" in fullk and second in fullk:
    a, b = fullk["decide"], fullk[second]
    fullk["decide_gather"] = {"kernel": "decide_gather", "time_ns": a["time_ns"] + b["time_ns"],
                              "dram_read": a["dram_read"] + b["dram_read"], "dram_write": a["dram_write"] + b["dram_write"]}

with open(os.path.join(OUT, f"ncu_launches_{tag}.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["schedule", "id", "kernel", "grid", "block", "time_ns", "dram_read_bytes", "dram_write_bytes"])
    for sch, ls in (("fused", lf), ("separate", lsep)):
        for d in ls:
            w.writerow([sch, d["id"], d["kernel"], d["grid"], d["block"], d["time_ns"], d["dram_read"], d["dram_write"]])
json.dump({"tag": tag, "step_fused": step_f, "step_separate": step_s, "dense": dense, "full": list(fullk.values())},
          open(os.path.join(OUT, f"ncu_full_{tag}.json"), "w"), indent=1)


def step_table(title, step):
    md = ["", f"## {title}", "", "| kernel | grid x block | time (us) | share | DRAM read (MB) | DRAM write (MB) |",
          "|---|---|---|---|---|---|"]
    tot = sum(d["time_ns"] or 0 for d in step) or 1
    for d in step:
        md.append(f"| {d['kernel']} | {d['grid']} x {d['block']} | {d['time_ns'] / 1e3:.1f} | "
                  f"{(d['time_ns'] or 0) / tot:.2f} | {(d['dram_read'] or 0) / 1e6:.1f} | {(d['dram_write'] or 0) / 1e6:.1f} |")
    md.append(f"| **total** | | **{tot / 1e3:.1f}** | | | |")
    return md


md = [f"# ncu summary ({tag})", "",
      f"Source: `tools/prof_r1c.sh {tag}` on one B200 (gpurun); `python tools/ncu_summary2.py {tag}`. Launch lists: "
      "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` of "
      "`bench.py --schedule fused|separate` (cold-cache, serialised: compare shares, not absolutes). Full capture: "
      "`ncu --set full --clock-control none`. Bench workload: N=128, 28x28x512, c_mid=128, S=4, r~0.5."]
md += step_table("Dynamic step, masker-fused schedule (the bench default at r = 0.5)", step_f)
md += step_table("Dynamic step, masker-separate schedule (north-star branch)", step_s)
md += step_table("Dense comparator (lasnet_dense_block, same kernels on every pixel)", dense)
md += ["", "## Full capture (per kernel)", "",
       "| kernel | time (us) | DRAM rd+wr (MB) | SM->L2 (MB) | DRAM % | L2 % | tensor % | smem LSU % | smem UMMA % | warps % | regs | top stalls |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for d in full_f + full_s:
    md.append(f"| {d['kernel']} | {d.get('time_ns', 0) / 1e3:.1f} | {(d.get('dram_read', 0) + d.get('dram_write', 0)) / 1e6:.1f} | "
              f"{d.get('l2_tex_sectors', 0) * 32 / 1e6:.0f} | {d.get('dram_pct', 0):.1f} | {d.get('l2_pct', 0):.1f} | "
              f"{d.get('tensor_pct', 0):.1f} | {d.get('smem_lsu_pct', 0):.1f} | {d.get('smem_tc_pct', 0):.1f} | "
              f"{d.get('warps_active_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
              + ", ".join(f"{k} {v:.0%}" for k, v in d["top_stalls"].items()) + " |")
open(os.path.join(OUT, f"ncu_summary_{tag}.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
