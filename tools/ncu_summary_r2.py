#!/usr/bin/env python
"""Summarise the round-2 ncu evidence (tools/prof_r2.sh) into profiles/ (committed).

Inputs (gpurun_out/):
  launches_bench_r2.csv           launch list of the bench command (first 400 launches)
  launches_net_r2.csv             every launch of one eager LAS-R101 forward with DRAM bytes
  net_once_names.json             the library's event names of that forward, in launch order
  launches_regnet_r2.csv, regnet_once_names.json   the same for LAS-RegNetY-800MF
  full_net_r2.ncu-rep, full_block_r2.ncu-rep       --set full captures
Outputs:
  profiles/ncu_launches_r2.csv    the launch lists (source column)
  profiles/ncu_full_r2.json       per event name: launches, mean time and DRAM bytes per launch over the
                                  forward (bench.py reads the dominant kernel's traffic here), and the
                                  --set full metrics of the captured kernels
  profiles/ncu_summary_r2.md      tables
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
GO = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
TWO = ("decide+ids", "decide+gather")  # one event name, two launches (unless the decide is cooperative)


def short(name):
    n = name.replace("lasnet::", "").replace(" ", "").replace("(int)", "").replace("(bool)", "")
    table = [("conv_tc_kernel<0,", "conv1_dyn"), ("conv_tc_kernel<1,", "conv2_dyn"), ("conv_tc_kernel<2,", "conv3_dyn"),
             ("conv_tc_kernel<3,", "conv1_dense"), ("conv_tc_kernel<4,", "conv2_dense"),
             ("conv_tc_kernel<5,", "conv3_dense"), ("conv_tc_kernel<6,", "conv1_mask"), ("conv_tc_kernel<7,", "stem_conv"),
             ("conv_tc_kernel<8,", "conv2_gather"),
             ("conv23_kernel<0", "conv23"), ("conv23_kernel<false", "conv23"),
             ("conv23_kernel<1", "conv23_dense"), ("conv23_kernel<true", "conv23_dense"),
             ("masker_compact_kernel", "mask_compact"), ("masker_kernel", "mask"), ("compact_kernel", "compact"),
             ("decide_kernel", "decide"), ("compact_gather_kernel", "compact_gather"),
             ("compact_idx_kernel", "compact_idx"), ("gconv_kernel", "gconv"), ("se_fc_kernel", "se_fc"),
             ("se_apply", "se_apply"), ("se_kernel", "se"), ("regnet_stem", "regnet_stem"),
             ("subsample", "subsample"), ("add_bias", "add_bias"), ("maxpool", "maxpool"), ("avgpool", "avgpool"),
             ("fc_kernel", "fc"), ("pack_stem", "stem_pack")]
    for k, v in table:
        if k in n:
            return v
    return name[:40]


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    per = OrderedDict()
    for r in csv.DictReader(lines[start:]):
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return [dict(id=int(k), kernel=short(v["name"]), grid=v["grid"], block=v["block"],
                 time_ns=v.get("gpu__time_duration.sum", 0.0), dram_read=v.get("dram__bytes_read.sum", 0.0),
                 dram_write=v.get("dram__bytes_write.sum", 0.0)) for k, v in per.items()]


def attribute(ls, names):
    """Walk the event names in order, consuming the ncu launches each covers (decide +
    ids / gather: two when the second kernel follows, else one); the head's avgpool+fc and
    the RegNet SE's pool + two GEMMs are one event each."""
    out = []
    i = 0
    for nm in names:
        take = 1
        if nm in TWO and i + 1 < len(ls) and ls[i + 1]["kernel"] in ("compact_idx", "compact_gather"):
            take = 2
        if nm == "head":
            take = 2
        if nm == "se":
            take = 3
        grp = ls[i:i + take]
        i += take
        out.append(dict(name=nm, kernels=[g["kernel"] for g in grp], time_ns=sum(g["time_ns"] for g in grp),
                        dram_read=sum(g["dram_read"] for g in grp), dram_write=sum(g["dram_write"] for g in grp)))
    return out, i


WANT = {
    "time_ns": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smem_lsu_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_tc_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread", "grid": "launch__grid_size",
}
SCALE = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full(rep):
    if not os.path.exists(rep):
        return []
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) < 3:
        return []
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


def per_name(attr):
    agg = OrderedDict()
    for a in attr:
        g = agg.setdefault(a["name"], {"kernel": a["name"], "launches": 0, "time_ns": 0.0, "dram_read": 0.0,
                                       "dram_write": 0.0})
        g["launches"] += 1
        g["time_ns"] += a["time_ns"]
        g["dram_read"] += a["dram_read"]
        g["dram_write"] += a["dram_write"]
    out = []
    for g in agg.values():
        k = g["launches"]
        out.append(dict(kernel=g["kernel"], launches=k, time_ns=g["time_ns"] / k, dram_read=g["dram_read"] / k,
                        dram_write=g["dram_write"] / k, total_time_ns=g["time_ns"]))
    return out


def main():
    rows = []
    res = {"tag": "r2"}
    md = ["# ncu summary (r2)", "",
          "Source: `tools/prof_r2.sh` on one B200 (gpurun), `python tools/ncu_summary_r2.py`. Launch lists: `ncu "
          "--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` "
          "(cold-cache, serialised launches: compare SHARES with bench.py's event timings, not absolutes). Full "
          "captures: `ncu --set full --clock-control none --import-source on`.", ""]
    for tag, csvf, namesf, title in (("net", "launches_net_r2.csv", "net_once_names.json",
                                      "LAS-ResNet-101 forward, N=256 224x224, r=0.5 (one eager forward)"),
                                     ("regnet", "launches_regnet_r2.csv", "regnet_once_names.json",
                                      "LAS-RegNetY-800MF forward, N=512 224x224, r=0.5 (one eager forward)")):
        p, pn = os.path.join(GO, csvf), os.path.join(GO, namesf)
        if not (os.path.exists(p) and os.path.exists(pn)):
            continue
        ls = launches(p)
        names = json.load(open(pn))["names"]
        attr, used = attribute(ls, names)
        for d in ls:
            rows.append([tag, d["id"], d["kernel"], d["grid"], d["block"], d["time_ns"], d["dram_read"], d["dram_write"]])
        pn_ = per_name(attr)
        res[tag] = pn_
        tot = sum(g["total_time_ns"] for g in pn_) or 1.0
        md += [f"## {title}", "", f"{len(ls)} launches ({used} attributed to {len(names)} library events).", "",
               "| kernel (event) | launches | mean us / launch | share of forward | DRAM rd+wr MB / launch | DRAM GB/s |",
               "|---|---|---|---|---|---|"]
        for g in sorted(pn_, key=lambda g: -g["total_time_ns"]):
            mb = (g["dram_read"] + g["dram_write"]) / 1e6
            md.append(f"| {g['kernel']} | {g['launches']} | {g['time_ns'] / 1e3:.1f} | {g['total_time_ns'] / tot:.3f} | "
                      f"{mb:.1f} | {mb * 1e6 / max(g['time_ns'], 1):.0f} |")
        md.append(f"| **total** | | | **{tot / 1e6:.3f} ms** | | |")
        md.append("")
    p = os.path.join(GO, "launches_bench_r2.csv")
    if os.path.exists(p):
        for d in launches(p):
            rows.append(["bench", d["id"], d["kernel"], d["grid"], d["block"], d["time_ns"], d["dram_read"],
                         d["dram_write"]])
    fulls = []
    for tag, rep in (("net stage 2-3", "full_net_r2.ncu-rep"), ("block", "full_block_r2.ncu-rep")):
        f = full(os.path.join(GO, rep))
        for d in f:
            d["capture"] = tag
        fulls += f
    # bench.py's ncu_traffic reads entries named by event: the forward's per-launch means first
    res["full"] = res.get("net", []) + fulls
    json.dump(res, open(os.path.join(OUT, "ncu_full_r2.json"), "w"), indent=1)
    with open(os.path.join(OUT, "ncu_launches_r2.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["source", "id", "kernel", "grid", "block", "time_ns", "dram_read_bytes", "dram_write_bytes"])
        w.writerows(rows)
    if fulls:
        md += ["## Full captures (`--set full`)", "",
               "| capture | kernel | grid | time (us) | DRAM rd+wr (MB) | DRAM % | L2 % | tensor % | smem LSU % | smem UMMA % | warps % | regs | top stalls |",
               "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        for d in fulls:
            md.append(f"| {d['capture']} | {d['kernel']} | {d.get('grid', 0):.0f} | {d.get('time_ns', 0) / 1e3:.1f} | "
                      f"{(d.get('dram_read', 0) + d.get('dram_write', 0)) / 1e6:.1f} | {d.get('dram_pct', 0):.1f} | "
                      f"{d.get('l2_pct', 0):.1f} | {d.get('tensor_pct', 0):.1f} | {d.get('smem_lsu_pct', 0):.1f} | "
                      f"{d.get('smem_tc_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
                      + ", ".join(f"{k} {v:.0%}" for k, v in d["top_stalls"].items()) + " |")
    open(os.path.join(OUT, "ncu_summary_r2.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
