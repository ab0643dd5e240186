"""Compact text summary of one-kernel ncu --set full captures (for profiles/).

    python tools/ncu_summary.py gpurun_out/r02f_tgram_tc.ncu-rep [...] > profiles/r02_ncu_full_summary.txt

Per report: duration, DRAM bytes (the `traffic` of the bench line), L2 / shared / tensor-pipe
utilisation, registers and occupancy from the raw page, and the warp-stall mix from the source
page (all samples).
"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared wavefronts %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__cycles_active.avg", "SM active cycles"),
]


def ncu(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summary(rep):
    rows = ncu(rep, "raw")
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}
    kname = vals[col["Kernel Name"]] if "Kernel Name" in col else "?"
    lines = [f"== {rep}", f"kernel: {re.sub(r'[(].*', '', kname)}"]
    for key, label in METRICS:
        if key in col:
            lines.append(f"  {label:28s} {vals[col[key]]} {units[col[key]]}".rstrip())
    src = ncu(rep, "source", ("--print-source", "sass"))
    if len(src) > 2:
        h = src[1]
        stall = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        agg = {c: 0 for c in stall}
        for r in src[2:]:
            for c in stall:
                v = r[h.index(c)]
                agg[c] += int(v) if v.isdigit() else 0
        tot = sum(agg.values()) or 1
        top = sorted(agg.items(), key=lambda x: -x[1])[:8]
        lines.append("  warp stalls (share of samples): " +
                     ", ".join(f"{c[6:]} {100.0 * v / tot:.1f}%" for c, v in top))
    return "\n".join(lines)


if __name__ == "__main__":
    print("\n\n".join(summary(r) for r in sys.argv[1:]))
