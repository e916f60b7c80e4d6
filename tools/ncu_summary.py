#!/usr/bin/env python
"""Summarise an ncu report (--set full) and/or a launch-list CSV for profiles/.

usage: ncu_summary.py REPORT.ncu-rep [--launches launches.csv] [--frames N --frame-bytes B] > out.md
Also writes the block kernel's DRAM bytes per frame to profiles/ncu_traffic.json when --workload is given."""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import collections

KEYS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy achieved)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__occupancy_limit_registers", "CTA limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active", "TMA pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, u, v in zip(rows[0], rows[1], r)})
    return res


def stalls(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = dict(zip(rows[0], rows[2]))
    st = {}
    for h, v in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
        if m:
            try:
                st[m.group(1)] = float(v)
            except ValueError:
                pass
    return sorted(st.items(), key=lambda kv: -kv[1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--launches")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--frame-bytes", type=int, default=0)
    ap.add_argument("--workload")
    ap.add_argument("--git", default=None, help="commit of the captured build (recorded with the traffic)")
    ap.add_argument("--date", default=None)
    a = ap.parse_args()
    ks = raw(a.report)
    for d in ks:
        name = d.get("Kernel Name", ("?",))[0]
        print("### %s\n" % name)
        print("| metric | value | unit |\n|---|---|---|")
        for k, label in KEYS:
            if k in d:
                print("| %s (`%s`) | %s | %s |" % (label, k, d[k][0], d[k][1]))
        if a.frames and "dram__bytes_read.sum" in d:
            def to_bytes(v, u):
                f = float(v.replace(",", ""))
                return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            rd = to_bytes(*d["dram__bytes_read.sum"])
            wr = to_bytes(*d["dram__bytes_write.sum"])
            print("\nDRAM traffic per launch: %.4g B (read %.4g + write %.4g) = %.4f x the algorithmic %d frames x %d B"
                  % (rd + wr, rd, wr, (rd + wr) / (a.frames * a.frame_bytes), a.frames, a.frame_bytes))
            if a.workload:
                p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                 "ncu_traffic.json")
                js = json.load(open(p)) if os.path.exists(p) else {}
                js[a.workload] = {"dram_bytes_per_frame": (rd + wr) / a.frames, "read": rd, "write": wr,
                                  "frames": a.frames, "report": os.path.basename(a.report), "git": a.git,
                                  "date": a.date}
                json.dump(js, open(p, "w"), indent=1)
        print("\nwarp stall reasons (warps per issue-active cycle):\n")
        for k, v in stalls(a.report)[:12]:
            print("- %s: %.3f" % (k, v))
        print()
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 5]
        hdr = rows[0]
        iK = hdr.index("Kernel Name")
        iV = hdr.index("Metric Value")
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for r in rows[1:]:
            try:
                v = float(r[iV].replace(",", ""))
            except ValueError:
                continue
            k = re.sub(r"\(.*", "", r[iK])
            tot[k] += v
            cnt[k] += 1
        T = sum(tot.values())
        print("### launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        print("| kernel | launches | total | share |\n|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            print("| %s | %d | %.4g | %.1f %% |" % (k, cnt[k], v, 100 * v / T))


if __name__ == "__main__":
    main()
