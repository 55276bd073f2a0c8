"""Summarise one kernel of an `ncu --set full` report (.ncu-rep) into markdown: the headline metrics, the
warp-stall breakdown (pc sampling) and the executed-instruction mix by opcode.
Usage: python tools/ncu_full_summary.py REPORT.ncu-rep [title] [command]"""
import collections
import csv
import io
import subprocess
import sys

HEADLINE = ["Duration", "Executed Instructions", "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy",
            "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size",
            "Grid Size", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "No Eligible",
            "Compute (SM) Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L1/TEX Hit Rate",
            "DRAM Throughput"]


def _csv(report, *args):
    out = subprocess.run(["ncu", "-i", report, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(report, title="", command=""):
    det = _csv(report, "--page", "details")
    hd = det[0]
    kn, mn, mu, mv = (hd.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    kernel = det[1][kn] if len(det) > 1 else "?"
    seen = {}
    for r in det[1:]:
        if len(r) > mv and r[mn] in HEADLINE and r[mn] not in seen:
            seen[r[mn]] = f"{r[mv]} {r[mu]}".strip()
    raw = _csv(report, "--page", "raw")
    h, units, v = raw[0], raw[1], raw[2]
    stalls = {}
    extra = {}
    for k, u, x in zip(h, units, v):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(x.replace(",", ""))
            except ValueError:
                pass
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                 "sm__pipe_tensor_op_umma_cycles_active.avg.pct_of_peak_sustained_elapsed"):
            extra[k] = f"{x} {u}".strip()
    src = _csv(report, "--page", "source", "--print-source", "sass")
    hh = src[1]
    ie, so = hh.index("Instructions Executed"), hh.index("Source")
    mix = collections.Counter()
    for r in src[2:]:
        toks = r[so].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        mix[op.split(".")[0]] += float(r[ie] or 0)
    tot = sum(mix.values()) or 1.0
    st = sum(stalls.values()) or 1.0
    out = [f"# {title}" if title else f"# ncu --set full: {kernel}", ""]
    if command:
        out += [f"Command: `{command}`", ""]
    out += [f"Kernel: `{kernel}`", "", "| metric | value |", "|---|---|"]
    out += [f"| {k} | {seen[k]} |" for k in HEADLINE if k in seen]
    out += [f"| {k} | {x} |" for k, x in extra.items()]
    out += ["", "Warp stalls (pc sampling, share of samples): " +
            ", ".join(f"{k} {x / st * 100:.1f}%" for k, x in sorted(stalls.items(), key=lambda a: -a[1]) if x / st > 0.02)]
    out += ["", "Instruction mix (share of executed warp instructions): " +
            ", ".join(f"{k} {x / tot * 100:.1f}%" for k, x in mix.most_common(16))]
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print(summarise(sys.argv[1], *(sys.argv[2:4])), end="")
