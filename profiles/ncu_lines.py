"""Per-source-line stall samples of an ncu report (compiled with -lineinfo).

    python profiles/ncu_lines.py gpurun_out/prof.ncu-rep [--top 30]

Prints the source lines with the most warp-stall samples and, per line, the dominant stall
reasons (ncu --page source --print-source cuda,sass).
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    idx = {h: i for i, h in enumerate(hdr)}
    samp = idx["Warp Stall Sampling (All Samples)"]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    lines, fname, total = [], None, 0
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        if not r or not r[0].isdigit() or len(r) <= samp:
            continue
        try:
            s = int(r[samp])
        except ValueError:
            continue
        total += s
        reasons = sorted(((int(r[idx[h]]) if r[idx[h]].isdigit() else 0, h[6:]) for h in stalls), reverse=True)[:3]
        lines.append((s, fname, r[0], r[1][:70], reasons))
    lines.sort(reverse=True)
    print(f"total samples {total}")
    for s, f, ln, src, rs in lines[:a.top]:
        rr = " ".join(f"{n}:{c}" for c, n in rs if c)
        print(f"{100.0 * s / max(total, 1):5.1f}%  {f}:{ln:5s} {src:70s} {rr}")


if __name__ == "__main__":
    main()
