#!/usr/bin/env python
"""Per-kernel DRAM traffic from an ncu --metrics CSV launch list (profiles/capture_r02.sh).

For each kernel name: mean gpu__time_duration, dram__bytes_read, dram__bytes_write and the L2
write bytes (lts__t_sectors_op_write x 32 B, informational: on B200 it reads ~1.5x the bytes a
kernel stores, the cross-die L2 traffic is counted too).  traffic = dram read + dram write as
the roofline contract defines it.  An output that fits in the 126 MB L2 can still be dirty in
L2 when its launch ends, so dram__bytes_write may undercount the write-back; dram read vs the
algorithmic input bytes is the re-read check.

    python tools/ncu_traffic.py gpurun_out/ncu_c2.csv --config c2 --alg-bytes 32149504 \
        [--merge profiles/r02_traffic.json]
"""
import argparse
import csv
import io
import json
import os


def parse(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), \
        hdr.index("Metric Unit")
    iid = hdr.index("ID")
    launches = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        unit = r[iu]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
                 "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3, "sector": 1}.get(unit, 1)
        launches.setdefault(r[iid], {"kernel": r[ik]})[r[im]] = v * scale
    return list(launches.values())


def summarize(launches):
    by = {}
    for l in launches:
        name = l["kernel"].split("(")[0].split("::")[-1]
        by.setdefault(name, []).append(l)
    out = {}
    for name, ls in by.items():
        def mean(k):
            vals = [x.get(k) for x in ls if x.get(k) is not None]
            return sum(vals) / len(vals) if vals else None
        rd, wr = mean("dram__bytes_read.sum"), mean("dram__bytes_write.sum")
        l2w = mean("lts__t_sectors_op_write.sum")
        l2w = l2w * 32 if l2w is not None else None
        out[name] = {"launches": len(ls), "us": mean("gpu__time_duration.sum"), "dram_read": rd, "dram_write": wr,
                     "l2_write_bytes": l2w,
                     "dram_pct": mean("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                     "tensor_pct": mean("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")}
        if rd is not None:
            out[name]["traffic"] = rd + (wr or 0)
            out[name]["total_traffic"] = (rd + (wr or 0)) * len(ls)
            out[name]["total_us"] = (out[name]["us"] or 0) * len(ls)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config")
    ap.add_argument("--kernel", default="", help="dominant kernel name substring")
    ap.add_argument("--alg-bytes", type=float, default=0)
    ap.add_argument("--merge")
    a = ap.parse_args()
    s = summarize(parse(a.csv))
    print(json.dumps(s, indent=1))
    if a.merge and a.config:
        cur = {}
        if os.path.exists(a.merge):
            cur = json.load(open(a.merge))
        dom = [k for k in s if a.kernel in k] or list(s)
        k = max(dom, key=lambda n: (s[n]["us"] or 0) * s[n]["launches"])
        e = dict(s[k], kernel=k, source=os.path.basename(a.csv), dram_bytes_per_launch=s[k].get("traffic"))
        if a.alg_bytes:
            e["algorithmic_bytes"] = a.alg_bytes
            e["traffic_over_algorithmic"] = round(e["traffic"] / a.alg_bytes, 3) if e.get("traffic") else None
        e["all_kernels_traffic"] = sum(v.get("total_traffic") or 0 for v in s.values())
        e["all_kernels_us"] = sum(v.get("total_us") or 0 for v in s.values())
        cur[a.config] = e
        json.dump(cur, open(a.merge, "w"), indent=1)


if __name__ == "__main__":
    main()
