"""Per-launch summary of an ncu --set full report (pipe utilisation, DRAM
traffic, stalls) -- the text committed under profiles/.

    python tools/ncu_summary.py <report.ncu-rep>
"""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_%"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_inst_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_thru_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_thru_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_thru_%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        print(f"== {short}  [ID {r[hdr.index('ID')]}]")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"   {label:15s} {r[i]} {units[i]}")
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda x: -float(x[1] or 0))[:5]
        print("   top stalls     " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={float(v):.2f}"
            for h, v in stalls))


if __name__ == "__main__":
    main(sys.argv[1])
