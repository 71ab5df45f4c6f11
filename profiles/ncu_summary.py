"""Summarise an ncu report: headline metrics + top SASS stall sites.

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [--top 20]
"""
import argparse
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:120])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {vals[i]:>14s} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        ia, isrc, ist = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = []
        for r in src[2:]:
            try:
                data.append((int(r[ist]), r[ia], r[isrc].strip()))
            except (ValueError, IndexError):
                pass
        tot = sum(d[0] for d in data) or 1
        print(f"top stall sites ({tot} samples):")
        for s, addr, txt in sorted(data, reverse=True)[: a.top]:
            print(f"  {100.0 * s / tot:5.1f}%  {addr[-5:]}  {txt[:90]}")


if __name__ == "__main__":
    main()
