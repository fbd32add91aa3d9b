"""Key metrics + SASS instruction mix of an ncu report (one kernel)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "smsp__inst_executed.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_op_red.sum", "lts__t_requests_op_red.sum",
        "smsp__sass_inst_executed_op_global_red.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_lg_throttle",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
        "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_drain", "smsp__pcsamp_warps_issue_stalled_no_instructions",
        "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
        "smsp__pcsamp_warps_issue_stalled_lsu_throttle" if False else "smsp__pcsamp_warps_issue_stalled_tex_throttle"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=25):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, units = raw[0], raw[1]
    print("kernel:", raw[2][h.index("Kernel Name")][:100])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:70s} {raw[2][i]:>16s} {units[i]}")
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source=sass"]))))
    hdr = rows[1]
    ai, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ops, st, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[ei].isdigit():
            continue
        ins = r[ai].strip().split()
        if not ins:
            continue
        op = (ins[1] if ins[0].startswith("@") else ins[0]).split(".")[0]
        ops[op] += int(r[ei])
        st[op] += int(r[si] or 0)
        tot += int(r[ei])
    print(f"  SASS instructions executed: {tot}")
    for op, n in ops.most_common(top):
        print(f"    {op:10s} {n:12d} {100 * n / tot:5.1f}%  stall-samples {st[op]}")


if __name__ == "__main__":
    main(sys.argv[1])
