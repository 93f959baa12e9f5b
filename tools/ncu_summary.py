#!/usr/bin/env python
"""Summarise an ncu report: key raw metrics, stall reasons, top SASS lines, instruction mix."""
import csv
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res = []
    for r in rows[2:]:
        res.append({h: (u, v) for h, u, v in zip(rows[0], rows[1], r)})
    return res


def main(rep, top=20):
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_sector_hit_rate.pct",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    for k in raw(rep):
        for key in keys:
            if key in k:
                print(f"{key:80s} {k[key][1]} {k[key][0]}")
        st = [(h, float(v[1].replace(',', ''))) for h, v in k.items()
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
              and v[1] not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        print("stalls per issue:", ", ".join(f"{h[34:-28]}={v:.2f}" for h, v in st[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    # the source page starts with a kernel-name line when the report holds one
    # kernel; find the header row by its columns instead of assuming row 1
    hi = next((i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r), None)
    if hi is None:
        print("(no SASS source page in this report)")
        return
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]

    def f(r, k):
        try:
            return float(r[idx[k]].replace(',', ''))
        except (ValueError, KeyError):
            return 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
    c = Counter()
    for r in data:
        toks = r[idx["Source"]].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        c[op.split(".")[0]] += f(r, "Instructions Executed")
    s = sum(c.values()) or 1
    print("dynamic instruction mix:", ", ".join(f"{k} {v / s * 100:.1f}%" for k, v in c.most_common(12)))
    print("top stall lines:")
    for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
        print(f"  {f(r, 'Warp Stall Sampling (All Samples)') / tot * 100:5.1f}%  {r[idx['Source']][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
