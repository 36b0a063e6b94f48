"""Summarise an ncu --set full report: key throughput metrics and stall
reasons per kernel.  usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
STALLS = ["long_scoreboard", "short_scoreboard", "mio_throttle", "lg_throttle", "barrier",
          "membar", "wait", "math_pipe_throttle", "not_selected", "selected", "sleeping",
          "branch_resolving", "no_instruction", "dispatch_stall", "drain", "misc", "tex_throttle"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print("==", r[col["Kernel Name"]][:90])
        for k in KEYS:
            if k in col:
                print(f"   {k:70s} {r[col[k]]:>14s} {units[col[k]]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in col:
                try:
                    st.append((float(r[col[k]]), s))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   stalls/issue:", ", ".join(f"{s}={v:.2f}" for v, s in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
