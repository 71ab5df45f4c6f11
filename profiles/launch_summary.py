"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file ...).

    python profiles/launch_summary.py gpurun_out/launches_c5.csv --steps 1 --title "config 5 ..."

Groups the launches of the LAST `--steps` bench steps by kernel name (the launch list is
cold-cache and serialised: shares of the step are meaningful, absolute times are not).
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--per-step", type=int, required=True, help="launches per bench step")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    launches = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1e3
        elif r[ui] == "msecond":
            v *= 1e6
        launches.append((r[ki], v))
    step = launches[-a.per_step:]
    tot = sum(v for _, v in step)
    g = collections.OrderedDict()
    for k, v in step:
        c, s = g.get(k, (0, 0.0))
        g[k] = (c + 1, s + v)
    print(f"# {a.title}, one step = {a.per_step} launches, ncu gpu__time_duration.sum "
          f"(--clock-control none; cold, serialised)")
    print(f"# total {tot:.1f} ns")
    for k, (c, s) in sorted(g.items(), key=lambda kv: -kv[1][1]):
        print(f"{s:12.1f} ns {100 * s / tot:5.1f}%  x {c:2d}  {k[:110]}")


if __name__ == "__main__":
    main()
