"""Summarise an ncu report into a committed text file (profiles/).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/rNN_name.txt "header line"
"""
import csv
import io
import subprocess
import sys


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, dst, header):
    lines = ["# " + h for h in header.split("\\n")]
    seen = set()
    det = page(rep, "details")
    h = det[0]
    isec, iname, iunit, ival = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    for row in det[1:]:
        if len(row) <= ival or not row[iname] or (row[isec], row[iname]) in seen:
            continue
        seen.add((row[isec], row[iname]))
        lines.append(f"{row[isec][:28]:28s} {row[iname][:52]:52s} {row[iunit]:12s} {row[ival]}")
    raw = page(rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    keep = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread")
    lines.append("# raw metrics")
    stalls = []
    for h, u, v in zip(hdr, units, vals):
        if h in keep:
            lines.append(f"{h} {u} {v}")
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    lines.append("# warp stall sampling (share of all samples)")
    for v, h in sorted(stalls, reverse=True)[:10]:
        lines.append(f"{v / tot * 100:6.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    open(dst, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
