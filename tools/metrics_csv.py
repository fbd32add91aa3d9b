"""metrics.csv in the reference's experiment layout --
`machine,policy,threshold,<RunMetrics>,grad_speedup,end_to_end_speedup`
(experiment.cpp:377-378, hwsim.cpp:515-527) -- populated from MEASURED ncu
counters of the B200 backward kernel instead of the simulator:

  total_cycles          sm__cycles_elapsed.max
  stalls_lsu            pc samples stalled on lg_throttle + mio_throttle
                        (the LSU / memory-input queue), scaled to cycles by
                        total_cycles / samples
  stalls_other          pc samples on long_scoreboard, same scaling
  atomic_requests_to_l2 lts__t_requests_op_red.sum
  core_instructions     sm__inst_executed.sum (warp instructions)
  core_fp_adds          smsp__sass_thread_inst_executed_op_fadd_pred_on.sum
  interconnect_packets  lts__t_sectors_op_red.sum (sectors of RED traffic)
  energy_proxy          10 * packets + 1 * (atomic requests + fp adds)
                        (hwsim.hpp:113-117 weights)
  grad_speedup          native time / this time
  end_to_end_speedup    Amdahl with grad_fraction (0.44: PAPER.md:1441)

    python tools/metrics_csv.py gpurun_out/thr_sweep_*.csv > metrics.csv
"""
import re
import sys

from threshold_sweep_summary import load

GRAD_FRACTION = 0.44
HEADER = ("machine,policy,threshold,total_cycles,stalls_lsu,stalls_other,atomic_requests_to_l2,"
          "core_instructions,core_fp_adds,interconnect_packets,energy_proxy,grad_speedup,"
          "end_to_end_speedup")


def main(paths):
    rows = []
    for p in paths:
        m = re.search(r"thr_sweep_(\w+?)_(\d+)\.csv", p)
        d = load(p)
        if not m or not d:
            continue
        rows.append((m.group(1), int(m.group(2)), d))
    order = {"native": 0, "sw_s": 1, "sw_b": 2, "cccl": 3}
    rows.sort(key=lambda r: (order.get(r[0], 9), r[1]))
    native = next((d for pol, _, d in rows if pol == "native"), None)
    print(HEADER)
    for pol, t, d in rows:
        cyc = d.get("sm__cycles_elapsed.max", 0.0)
        samples = d.get("smsp__pcsamp_sample_count", 0.0) or 1.0
        lsu = d.get("smsp__pcsamp_warps_issue_stalled_lg_throttle", 0.0) + \
            d.get("smsp__pcsamp_warps_issue_stalled_mio_throttle", 0.0)
        other = d.get("smsp__pcsamp_warps_issue_stalled_long_scoreboard", 0.0)
        reqs = d.get("lts__t_requests_op_red.sum", 0.0)
        fadd = d.get("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", 0.0)
        pk = d.get("lts__t_sectors_op_red.sum", 0.0)
        ms = d.get("gpu__time_duration.sum", float("nan"))
        gs = native["gpu__time_duration.sum"] / ms if native else float("nan")
        e2e = 1.0 / (GRAD_FRACTION / gs + (1.0 - GRAD_FRACTION))
        thr = str(t) if pol in ("sw_s", "sw_b") else "-"
        print(f"b200,{pol},{thr},{int(cyc)},{int(lsu * cyc / samples)},{int(other * cyc / samples)},"
              f"{int(reqs)},{int(d.get('sm__inst_executed.sum', 0))},{int(fadd)},{int(pk)},"
              f"{10.0 * pk + reqs + fadd:.6g},{gs:.6g},{e2e:.6g}")


if __name__ == "__main__":
    sys.path.insert(0, __file__.rsplit("/", 1)[0])
    main(sys.argv[1:])
