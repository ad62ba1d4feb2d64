"""Per-CUDA-source-line view of one kernel in an .ncu-rep (needs -lineinfo +
--import-source): stall samples and warp instructions executed per line.

  python tools/ncu_lines.py report.ncu-rep [--kernel 0] [--top 40]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(a.kernel), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    lo, hi = 0, len(rows)  # one launch; sections per source file ("File Path")
    agg = {}
    hdr = None
    fname = "?"
    for r in rows[lo:hi]:
        if not r:
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if hdr is None or not r[0] or len(r) != len(hdr):
            continue
        iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        key = (fname, int(r[0]))
        s, e = float(r[iss] or 0), float(r[iex] or 0)
        p = agg.setdefault(key, [0.0, 0.0, r[1]])
        p[0] += s
        p[1] += e
    ts = sum(v[0] for v in agg.values()) or 1
    te = sum(v[1] for v in agg.values()) or 1
    print(f"kernel {a.kernel}: {te:.4g} warp instructions, {ts:.0f} stall samples")
    for (f, ln), (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
        print(f"  {f}:{ln:<5d} stall {100 * s / ts:5.1f}%  inst {100 * e / te:5.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    main()
