"""Summarise one kernel of an .ncu-rep: key throughput metrics, stall reasons, top stalled SASS lines.

  python tools/ncu_brief.py report.ncu-rep [--top 20]
"""
import argparse
import csv
import io
import subprocess

KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.per_cycle_active",
        "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=20)
    ap.add_argument("--kernel", type=int, default=0, help="index of the launch in the report")
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "raw", "--csv"))))
    h, units, v = rows[0], rows[1], rows[2 + a.kernel]
    print("kernel:", v[h.index("Kernel Name")][:100])
    for k in KEYS:
        if k in h:
            print(f"  {k} = {v[h.index(k)]} {units[h.index(k)]}")
    st = [(k, float(v[i] or 0)) for i, k in enumerate(h)
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    print("  stall samples:")
    for k, x in sorted(st, key=lambda t: -t[1])[:8]:
        print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {100 * x / tot:5.1f}%")
    src = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "source", "--csv", "--print-source", "sass"))))
    starts = [i for i, r in enumerate(src) if r and r[0] == "Kernel Name"] + [len(src)]
    sect = src[starts[a.kernel] + 1: starts[a.kernel + 1]]
    hh, body = sect[0], [r for r in sect[1:] if len(r) == len(sect[0])]
    ia, isrc = hh.index("Address"), hh.index("Source")
    iss, iex = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    tot = sum(float(r[iss] or 0) for r in body) or 1
    print(f"  top stalled SASS ({len(body)} instructions):")
    for r in sorted(body, key=lambda r: -float(r[iss] or 0))[: a.top]:
        print(f"    {r[ia][-5:]} {100 * float(r[iss] or 0) / tot:5.2f}%  {r[isrc].strip()[:70]}")


if __name__ == "__main__":
    main()
